"""Measurement of the widened rows beside the per-frame path:
init-time pair geometry, feature refinement and the quality metrics, device
vs the CPU oracle on the same inputs.  Prints one JSON object.

  python scripts/bench_widened.py [c2|c4]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import bench  # noqa: E402
import oracle as O  # noqa: E402
import paper_2308_09209_b200 as pb  # noqa: E402


def best_of(fn, n=3):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "c2"
    wl = bench.WORKLOADS[key]
    sc = bench.build_scene(wl, 1)
    cfg = sc.config()
    nv = wl["views"]
    first = [sc.render_view(v, 0) for v in range(nv)]
    threads = bench.cpu_cores()
    c = sc.config_c()
    cams = [(c.cams[v].fx, c.cams[v].fy, c.cams[v].cx, c.cams[v].cy, list(c.cams[v].rotation),
             list(c.cams[v].translation)) for v in range(nv)]
    sizes = [(wl["width"], wl["height"])] * nv
    out = {"workload": wl["desc"], "config_key": key, "cpu_threads": threads}

    # init-time geometry (rebuild_pair_geometry) + context build: device vs
    # oracle (the first call also loads the CUDA module: reported apart)
    t0 = time.perf_counter()
    pb.initialize(cfg, first).close()
    out["first_init_s"] = round(time.perf_counter() - t0, 3)

    def init_only(c_):
        st = pb.initialize(c_, first)
        t = time.perf_counter()
        st.close()
        return t

    def timed_init(c_, n=5):
        ts = []
        for _ in range(n):
            t0 = time.perf_counter()
            t1 = init_only(c_)
            ts.append(t1 - t0)
        return min(ts)

    out["init_geometry_s"] = round(timed_init(cfg), 4)
    ocfg = O.make_config(nv, c.reference, sizes, cams, threads=threads, topology=c.topology)
    out["init_geometry_oracle_s"] = round(best_of(lambda: O.OracleState(ocfg).close(), 1), 4)

    # feature refinement (initialize with the first frames)
    cfg.refine.enabled = True
    out["init_refine_s"] = round(timed_init(cfg), 4)
    ocfg_r = O.make_config(nv, c.reference, sizes, cams, threads=threads, topology=c.topology,
                           refine=True)
    data = [f.data for f in first]
    out["init_refine_oracle_s"] = round(
        best_of(lambda: O.OracleState(ocfg_r, data).close(), 1), 4)
    cfg.refine.enabled = False

    # quality metrics: PSNR / SSIM of two 1080p frames, pair quality of a frame
    a, b = first[0], first[1]
    pb.psnr(a, b)
    out["psnr_s"] = round(best_of(lambda: pb.psnr(a, b)), 5)
    out["ssim_s"] = round(best_of(lambda: pb.ssim(a, b)), 5)
    out["psnr_oracle_s"] = round(best_of(lambda: O.psnr(a.data, None, b.data, None), 1), 5)
    out["ssim_oracle_s"] = round(best_of(lambda: O.ssim(a.data, None, b.data, None), 1), 5)
    state = pb.initialize(cfg, first)
    pb.process_frame(state, first)
    state.pair_quality(0)
    out["pair_quality_s"] = round(best_of(lambda: state.pair_quality(0)), 5)
    state.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
