"""Generate tests/golden/oracle_small.json: SHA-256 checksums of the CPU
oracle's outputs (panorama RGB + mask, colour matrices, both flow fields of
every pair, thresholds) for small fixed synthetic scenes.  The oracle is the
restatement of the reference path (oracle/stitch_oracle.c, pinned to the
reference's own test vectors in tests/test_oracle_pins.py); these fixtures
freeze its outputs so that (1) any change to the oracle is caught on CPU and
(2) the B200 path is checked against them without re-running the oracle.
Usage: python tests/golden/make_golden.py  (rewrites the JSON)."""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import paper_2308_09209_b200 as pb  # noqa: E402
from tests.helpers import frames_at, oracle_config, scene  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "oracle_small.json")

# (name, scene kwargs, config kwargs, frames)
CASES = [
    ("two_view_c1_like", dict(views=2, width=160, height=120, frames=3,
                              casts=[(1, 1, 1), (0.85, 1.0, 1.1)]), {}, 3),
    ("three_view_star_flicker", dict(views=3, width=200, height=150, frames=4,
                                     casts=[(0.9, 1, 1), (1, 1, 1), (1, 0.95, 1.1)],
                                     flicker=[pb.FlickerEvent(frame=2, view=1,
                                                              gains=(1.2, 1.1, 0.9))]), {}, 4),
    ("four_view_chain_window1", dict(views=4, width=160, height=96, frames=2, focal_scale=1.03,
                                     casts=[(1, 1, 1), (0.9, 1, 1.05), (1.05, 1, 0.95),
                                            (1, 0.92, 1)]), dict(window=1), 2),
]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def case_digest(sc, ckw, frames):
    ost = O.OracleState(oracle_config(sc, **ckw))
    out = {"canvas": list(ost.canvas), "pairs": ost.n_pairs(), "frames": []}
    try:
        for t in range(frames):
            data, mask, rep = ost.process([f.data for f in frames_at(sc, t)])
            fr = {"pano_rgb": sha(data), "pano_mask": sha(mask),
                  "m": [sha(np.array(rep.m[k][:], np.float64)) for k in range(ost.n_pairs())],
                  "rank_deficient": [int(rep.rank_deficient[k]) for k in range(ost.n_pairs())],
                  "m1": list(rep.threshold_m1), "m2": list(rep.threshold_m2),
                  "flows": []}
            for k in range(ost.n_pairs()):
                for d in range(2):
                    u, v = ost.last_flow(k, d)
                    fr["flows"].append(sha(np.stack([u, v])))
            out["frames"].append(fr)
    finally:
        ost.close()
    return out


def main():
    doc = {"generator": "tests/golden/make_golden.py", "cases": {}}
    for name, skw, ckw, frames in CASES:
        doc["cases"][name] = case_digest(scene(**skw), ckw, frames)
    with open(OUT, "w") as f:
        json.dump(doc, f, indent=1)
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
