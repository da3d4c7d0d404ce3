"""Full-size parity at the BASELINE.json configurations: the B200 path against
the CPU oracle on the bench's own synthetic inputs (bench.WORKLOADS /
bench.build_scene), stage by stage, with a max-abs-diff report.

Used by tests/test_gpu_fullsize.py (asserts the contract tolerances and the
bit-exact expectation) and scripts/parity_report.py (writes the per-stage,
per-frame report committed under profiles/).  The oracle is the checker here;
nothing in the product path imports this module.
"""
from __future__ import annotations

import os
import time

import numpy as np

import bench
import oracle as O
import paper_2308_09209_b200 as pb
from tests.helpers import frames_at, oracle_config, product_config

# frames checked per config: C2 spans the flicker event (frame 5) so the 3D-M
# window and the threshold history are exercised at full size
FRAMES = {"c1": 8, "c2": 7, "c3": 3, "c4": 2}


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _flow(state, k, d, shape):
    import ctypes as C

    from paper_2308_09209_b200 import _abi

    u = np.zeros(shape, np.float32)
    v = np.zeros(shape, np.float32)
    pb.pipeline.check(_abi.load().stitch_b200_debug_flow(state.handle, k, d,
                                                         u.ctypes.data_as(C.c_void_p),
                                                         v.ctypes.data_as(C.c_void_p)))
    return u, v


def frame_diffs(state, ost, frames):
    """Process one frame on both paths; return the max-abs-diff per stage."""
    res = pb.process_frame(state, frames)
    odata, omask, orep = ost.process([f.data for f in frames])
    rep = res.report
    m_rel = 0.0
    rank_ok = True
    for k in range(len(state.pairs)):
        m_ref = np.array(orep.m[k][:]).reshape(3, 3)
        m = rep.color_matrices[k]
        den = np.maximum(np.abs(m_ref), 1e-300)
        m_rel = max(m_rel, float((np.abs(m - m_ref) / den).max()))
        rank_ok &= rep.rank_deficient[k] == bool(orep.rank_deficient[k])
    flow = 0.0
    for k, p in enumerate(state.pairs):
        shape = (p.bounds[3] - p.bounds[1], p.bounds[2] - p.bounds[0])
        for d in range(2):
            u, v = _flow(state, k, d, shape)
            ou, ov = ost.last_flow(k, d)
            flow = max(flow, float(np.abs(u - ou).max()), float(np.abs(v - ov).max()))
    pano = int(np.abs(res.panorama.data.astype(np.int32) - odata.astype(np.int32)).max())
    return {
        "color_matrix_max_rel": m_rel,
        "rank_flags_equal": bool(rank_ok),
        "flow_max_abs_px": flow,
        "thresholds_equal": (rep.balanced == bool(orep.balanced)
                             and rep.threshold_m1 == list(orep.threshold_m1)
                             and rep.threshold_m2 == list(orep.threshold_m2)),
        "frame_index_equal": rep.frame_index == orep.frame_index,
        "panorama_max_abs_lsb": pano,
        "mask_equal": bool((res.panorama.mask == omask).all()),
    }


def run_config(key: str, frames: int | None = None, seed: int = 1, refine: bool | None = None):
    """Initialise both paths on the bench's inputs for `key` and compare
    `frames` frames; returns (geometry_equal, per-frame diff dicts, info).
    refine (default: as bench.py, i.e. on for the planar rigs, off for the
    360-degree ring) runs the feature refinement at initialize on both paths."""
    wl = bench.WORKLOADS[key]
    sc = bench.build_scene(wl, seed)
    n = frames or FRAMES[key]
    threads = host_threads()
    if refine is None:
        refine = wl.get("rig", "auto") != "ring"
    t0 = time.perf_counter()
    first = frames_at(sc, 0)
    state = pb.initialize(product_config(sc, refine=refine, seed=sc.spec.seed), first)
    ost = O.OracleState(oracle_config(sc, threads=threads, refine=refine, seed=sc.spec.seed),
                        first_frames=[f.data for f in first] if refine else None)
    geom = state.canvas == ost.canvas and len(state.pairs) == ost.n_pairs()
    for v in range(sc.spec.views):
        _, inv = ost.maps(v)
        geom &= bool(np.array_equal(state.inv_map(v), inv))
    for k, p in enumerate(state.pairs):
        view, partner, bounds = ost.pair(k)
        geom &= (p.view, p.partner, p.bounds) == (view, partner, bounds)
        geom &= bool(np.array_equal(p.theta_i, ost.pair_weights(k)))
    per_frame = []
    try:
        for t in range(n):
            per_frame.append(frame_diffs(state, ost, frames_at(sc, t)))
    finally:
        info = {"config": key, "workload": wl["desc"], "cameras": wl["views"], "refine": refine,
                "camera_size": [wl["width"], wl["height"]], "canvas": list(state.canvas[:2]),
                "pairs": len(state.pairs), "frames": n, "oracle_threads": threads,
                "seconds": round(time.perf_counter() - t0, 1)}
        state.close()
        ost.close()
    return bool(geom), per_frame, info
