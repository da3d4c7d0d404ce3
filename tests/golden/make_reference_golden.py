"""Generate tests/golden/reference_small.json from THE REFERENCE ITSELF.

Runs the unmodified reference sources (/root/reference/proj/src, compiled by
oracle/ref/Makefile into oracle/_ref/libstitch_ref.so, bound by
oracle/reference.py) through their own public API -- stitch::SynthScene,
stitch::initialize, stitch::process_frame (pipeline.hpp:73-92) and the
per-op functions warp_frame / dense_flow (geometry.hpp:63, flow.hpp:40) -- and
records SHA-256 digests of every output:

* per case: canvas size/offset, the pairs (view, overlap bounds), theta_i/j;
* per frame: panorama RGB + mask, every colour matrix (float64 bytes), rank
  flags, balance thresholds m1/m2;
* per op (C1 first frame): each view's warp onto the canvas (RGB + mask), and
  both flow fields of the overlap crops.

The digests are reference data: tests/test_ref_pin.py checks that the oracle
(oracle/stitch_oracle.c) reproduces them on CPU, and that the B200 path does
on the GPU, neither consulting the reference at test time (it is absent on the
GPU box).  The inputs are the reference's own renderer; the test also checks
that the repo's SynthScene renders the same bytes.

Usage (needs /root/reference): python tests/golden/make_reference_golden.py
"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from tests.golden.masks import case_masks  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_small.json")

OBJ = dict(enabled=True, half_size=40.0, velocity=(3.0, 1.0))
FLICKER = [dict(frame=3, view=1, gains=(1.25, 1.1, 0.9))]

# (name, scene kwargs (reference SynthSpec terms), StitchConfig overrides, frames)
CASES = [
    # C1 = BASELINE configs[0]: 2 x 640x480, 30 frames, the reference's defaults
    # (refinement on, window 3, lambda 0.05, gamma 1.5/1.5, targets 0/255).
    ("c1_defaults", dict(views=2, width=640, height=480, frames=30,
                         casts=[(1, 1, 1), (0.85, 1.0, 1.1)], obj=OBJ, flicker=FLICKER),
     dict(refine_enabled=1), 30),
    # C1 without refinement (the camera homographies as given).
    ("c1_norefine", dict(views=2, width=640, height=480, frames=6,
                         casts=[(1, 1, 1), (0.85, 1.0, 1.1)], obj=OBJ, flicker=FLICKER),
     dict(refine_enabled=0), 6),
    # non-default balancing: gammas, targets, lambda; window 2, cross weighting
    ("balance_a", dict(views=2, width=320, height=240, frames=5,
                       casts=[(1, 1, 1), (0.8, 1.0, 1.15)], obj=OBJ, flicker=FLICKER),
     dict(refine_enabled=0, gamma_dark=2.2, gamma_bright=0.45, target_black=16,
          target_white=235, lam=0.1, window_capacity=2, fuse_weighting=1), 5),
    ("balance_b", dict(views=2, width=320, height=240, frames=4,
                       casts=[(1.1, 1, 0.9), (0.8, 1.0, 1.15)], obj=OBJ),
     dict(refine_enabled=0, gamma_dark=0.45, gamma_bright=3.0, target_black=40,
          target_white=200, lam=0.02, window_capacity=1), 4),
    ("balance_c", dict(views=3, width=320, height=240, frames=4,
                       casts=[(0.9, 1, 1), (1, 1, 1), (1, 0.95, 1.1)], obj=OBJ),
     dict(refine_enabled=0, gamma_dark=1.0, gamma_bright=1.0, target_black=0,
          target_white=255, lam=0.25), 4),
    # 3-view star (the reference's largest rig), refinement on, flicker.
    ("star3_refine", dict(views=3, width=320, height=240, frames=5,
                          casts=[(0.9, 1, 1), (1, 1, 1), (1, 0.95, 1.1)], obj=OBJ,
                          flicker=[dict(frame=2, view=2, gains=(1.2, 1.1, 0.9))]),
     dict(refine_enabled=1), 5),
    # perturbed intrinsics ("coarse homographies"), flow options changed
    ("star3_perturbed_flow", dict(views=3, width=320, height=240, frames=3, focal_scale=1.03,
                                  principal_px=4.0, obj=OBJ),
     dict(refine_enabled=0, levels=3, iterations=20, smoothness=10.0), 3),
    # sweeps = iterations / 5 by integer division (flow.cpp:79-80): 23 -> 4 sweeps per
    # warp iteration; two pyramid levels, a smaller smoothness
    ("flow_iter23_levels2", dict(views=2, width=320, height=240, frames=3, obj=OBJ,
                                 casts=[(1, 1, 1), (0.9, 1.05, 1.0)]),
     dict(refine_enabled=0, levels=2, iterations=23, smoothness=7.5), 3),
    # narrow and wide overlaps (geometry, bounds, chamfer weights), seed 7
    ("narrow_overlap", dict(seed=7, views=2, width=320, height=240, frames=3, overlap=0.12,
                            obj=OBJ, casts=[(1, 1, 1), (1.1, 0.95, 0.9)]),
     dict(refine_enabled=1), 3),
    ("wide_overlap", dict(seed=7, views=3, width=320, height=240, frames=3, overlap=0.6,
                          obj=OBJ, casts=[(0.95, 1, 1), (1, 1, 1), (1, 1.05, 0.92)]),
     dict(refine_enabled=1, window_capacity=1, fuse_weighting=1), 3),
    # small frames: the pyramid stop rule checks the previous level (flow.cpp:153)
    ("small_frames", dict(seed=3, views=2, width=96, height=72, frames=4, obj=dict(
        enabled=True, half_size=12.0, velocity=(2.0, 1.0)), casts=[(1, 1, 1), (0.8, 1, 1.2)]),
     dict(refine_enabled=0), 4),
    # MASKED INPUTS (Frame::mask, e.g. PNG alpha): the sampler skips masked taps
    # (frame.cpp:95-104) and the pair geometry follows the masked first
    # frames (pipeline.cpp:181-205); C1 with refinement, masks on both views
    ("c1_masked", dict(views=2, width=640, height=480, frames=6, obj=OBJ, flicker=FLICKER,
                       casts=[(1, 1, 1), (0.85, 1.0, 1.1)],
                       masks=dict(seed=11, views=[0, 1])),
     dict(refine_enabled=1), 6),
    # 3-view star, masks on two views, one frame unmasked (mixed inputs)
    ("star3_masked_mixed", dict(views=3, width=320, height=240, frames=4, obj=OBJ,
                                casts=[(0.9, 1, 1), (1, 1, 1), (1, 0.95, 1.1)],
                                masks=dict(seed=12, views=[0, 2], skip_frames=[2])),
     dict(refine_enabled=0), 4),
    # full HD: the reference's own 3 x 1080p star rig (canvas
    # 7082 x 2111, overlaps 713 x 1080), refinement on, flicker -- the sizes
    # the bench runs at, pinned to the reference itself
    ("star3_1080p", dict(views=3, width=1920, height=1080, frames=3, obj=dict(
        enabled=True, half_size=120.0, velocity=(9.0, 3.0)),
                         casts=[(0.9, 1, 1), (1, 1, 1), (1, 0.95, 1.1)],
                         flicker=[dict(frame=1, view=0, gains=(1.2, 1.1, 0.9))]),
     dict(refine_enabled=1), 3),
    # perturbed principal point refined away, 5 frames
    ("principal_refine", dict(seed=5, views=3, width=320, height=240, frames=5,
                              focal_scale=1.02, principal_px=6.0, obj=OBJ,
                              casts=[(1, 1, 1), (0.9, 1, 1.05), (1.05, 0.97, 1)]),
     dict(refine_enabled=1, lam=0.08), 5),
]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def frame_masks(skw, t):
    spec = skw.get("masks")
    if spec is None:
        return None
    return [case_masks(spec, v, t, skw["width"], skw["height"]) for v in range(skw["views"])]


def run_case(R, skw, okw, frames, threads=8):
    skw = dict(skw)
    mspec = skw.pop("masks", None)
    sc = R.Scene(**skw)
    skw["masks"] = mspec
    first = [sc.render(v, 0) for v in range(sc.views)]
    st = R.State(sc, R.default_opts(threads=threads, **okw), first, frame_masks(skw, 0))
    out = {"canvas": list(st.canvas), "reference_view": sc.reference,
           "input_digest": [sha(f) for f in first], "pairs": []}
    if mspec is not None:
        out["mask_digest"] = [[None if m is None else sha(m) for m in frame_masks(skw, t)]
                              for t in range(frames)]
    for k in range(st.n_pairs()):
        v, b, warn = st.pair(k)
        ti, tj = st.pair_weights(k)
        out["pairs"].append({"view": v, "bounds": list(b), "refine_warning": warn,
                             "theta_i": sha(ti), "theta_j": sha(tj)})
    out["maps"] = [sha(st.maps(v)[0]) for v in range(sc.views)]
    out["map_values"] = [st.maps(v)[0].tolist() for v in range(sc.views)]
    out["frames"] = []
    for t in range(frames):
        fr = [sc.render(v, t) for v in range(sc.views)]
        rgb, mask, rep = st.process(fr, frame_masks(skw, t))
        out["frames"].append({
            "pano_rgb": sha(rgb), "pano_mask": sha(mask),
            "m": [sha(np.array(rep.m[k][:], np.float64)) for k in range(rep.n_pairs)],
            "rank_deficient": [int(rep.rank_deficient[k]) for k in range(rep.n_pairs)],
            "m1": list(rep.m1), "m2": list(rep.m2)})
    return sc, st, out


def op_digests(R, sc, st, levels=4, iterations=50, smoothness=15.0):
    """warp_frame of every view, dense_flow of every pair's raw overlap crops."""
    cw, ch, ox, oy = st.canvas
    fr = [sc.render(v, 0) for v in range(sc.views)]
    warped = [R.warp_frame(fr[v], None, st.maps(v)[0], cw, ch, ox, oy) for v in range(sc.views)]
    ops = {"warp": [[sha(w[0]), sha(w[1])] for w in warped], "flow": []}
    ref = sc.reference
    for k in range(st.n_pairs()):
        v, (x0, y0, x1, y1), _ = st.pair(k)
        ci = (warped[v][0][y0:y1, x0:x1], warped[v][1][y0:y1, x0:x1])
        cj = (warped[ref][0][y0:y1, x0:x1], warped[ref][1][y0:y1, x0:x1])
        uij = R.dense_flow(ci[0], ci[1], cj[0], cj[1], levels, iterations, smoothness, 8)
        uji = R.dense_flow(cj[0], cj[1], ci[0], ci[1], levels, iterations, smoothness, 8)
        ops["flow"].append([sha(np.stack(uij)), sha(np.stack(uji))])
    return ops


def main():
    import oracle.reference as R

    doc = {"generator": "tests/golden/make_reference_golden.py",
           "source": "unmodified /root/reference/proj/src via oracle/_ref/libstitch_ref.so "
                     "(Eigen-subset shim oracle/ref/eigen_shim)",
           "cases": {}}
    for name, skw, okw, frames in CASES:
        t0 = time.time()
        sc, st, out = run_case(R, skw, okw, frames)
        if name in ("c1_defaults", "star3_refine", "star3_1080p"):
            out["ops"] = op_digests(R, sc, st)
        doc["cases"][name] = {"scene": skw, "opts": okw, "n_frames": frames, **out}
        print(f"{name}: {frames} frames in {time.time() - t0:.1f} s", flush=True)
    with open(OUT, "w") as f:
        json.dump(doc, f, indent=1)
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
