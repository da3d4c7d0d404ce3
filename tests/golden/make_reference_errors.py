"""Generate tests/golden/reference_errors.json from THE REFERENCE ITSELF:
the error behaviour of stitch::initialize / stitch::process_frame on masked
inputs that warp to nothing.

warp_frame throws EmptyProjection when no canvas pixel of a view is valid
(geometry.cpp:79).  process_frame warps every view first (pipeline.cpp:
270-277), so such a frame fails before any state changes: the 3D-M windows,
the threshold history and the frame counter stay as they were and the next
frame continues from there.  initialize warps every first frame in
rebuild_pair_geometry (pipeline.cpp:181-188) before it looks at overlaps, so
a fully masked first frame is EmptyProjection, not NoOverlap.

Per case: the init error code (ErrorCode, types.hpp:9-27), or the canvas and
per frame either {"error": code} or the digests of make_reference_golden.py.
Usage (needs /root/reference): python tests/golden/make_reference_errors.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from tests.golden.make_reference_golden import OBJ, frame_masks, sha  # noqa: E402,I100

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_errors.json")

CASTS2 = [(1, 1, 1), (0.85, 1.0, 1.1)]
CASTS3 = [(0.9, 1, 1), (1, 1, 1), (1, 0.95, 1.1)]

# (name, scene kwargs, StitchConfig overrides, frames)
CASES = [
    # frames 2 (view 1) and 4 (the reference view) fully masked: those frames
    # fail, the others match a run that never saw them
    ("frame_empty", dict(views=2, width=320, height=240, frames=6, obj=OBJ, casts=CASTS2,
                         masks=dict(seed=21, views=[0, 1], empty=[[2, 1], [4, 0]])),
     dict(refine_enabled=1), 6),
    ("star3_frame_empty", dict(views=3, width=320, height=240, frames=4, obj=OBJ, casts=CASTS3,
                               masks=dict(seed=22, views=[2], empty=[[1, 2]])),
     dict(refine_enabled=0, window_capacity=2), 4),
    # a fully masked first frame: initialize fails
    ("first_frame_empty", dict(views=2, width=320, height=240, frames=1, obj=OBJ, casts=CASTS2,
                               masks=dict(seed=23, views=[1], empty=[[0, 1]])),
     dict(refine_enabled=1), 1),
    ("first_frame_empty_norefine", dict(views=3, width=320, height=240, frames=1, obj=OBJ,
                                        casts=CASTS3,
                                        masks=dict(seed=24, views=[0], empty=[[0, 0]])),
     dict(refine_enabled=0), 1),
]


def run_case(R, skw, okw, frames, threads=8):
    skw = dict(skw)
    mspec = skw.pop("masks")
    sc = R.Scene(**skw)
    skw["masks"] = mspec
    first = [sc.render(v, 0) for v in range(sc.views)]
    try:
        st = R.State(sc, R.default_opts(threads=threads, **okw), first, frame_masks(skw, 0))
    except R.RefError as e:
        return {"init_error": e.code}
    out = {"canvas": list(st.canvas), "frames": []}
    for t in range(frames):
        fr = [sc.render(v, t) for v in range(sc.views)]
        try:
            rgb, mask, rep = st.process(fr, frame_masks(skw, t))
        except R.RefError as e:
            out["frames"].append({"error": e.code})
            continue
        out["frames"].append({
            "pano_rgb": sha(rgb), "pano_mask": sha(mask),
            "m": [sha(np.array(rep.m[k][:], np.float64)) for k in range(rep.n_pairs)],
            "rank_deficient": [int(rep.rank_deficient[k]) for k in range(rep.n_pairs)],
            "m1": list(rep.m1), "m2": list(rep.m2)})
    st.close()
    return out


def main():
    import oracle.reference as R

    doc = {"generator": "tests/golden/make_reference_errors.py",
           "source": "unmodified /root/reference/proj/src via oracle/_ref/libstitch_ref.so",
           "error_codes": "stitch::ErrorCode (types.hpp:9-27), EmptyProjection = 10",
           "cases": {}}
    for name, skw, okw, frames in CASES:
        out = run_case(R, skw, okw, frames)
        doc["cases"][name] = {"scene": skw, "opts": okw, "n_frames": frames, **out}
        print(name, out.get("init_error"), [f.get("error") for f in out.get("frames", [])])
    with open(OUT, "w") as f:
        json.dump(doc, f, indent=1)
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
