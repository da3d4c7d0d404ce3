"""Where the synchronous host-buffer call's time goes at C2 (one B200):
stitch_b200_process with pinned / pageable inputs and outputs, and the host
memcpy rate.  Usage: python scripts/sync_breakdown.py [reps]"""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2308_09209_b200 as pb  # noqa: E402
from paper_2308_09209_b200 import _abi  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    lib = _abi.load()
    wl = bench.WORKLOADS["c2"]
    sc = bench.build_scene(wl, seed=1)
    cfg = sc.config()
    nv = wl["views"]
    fb = wl["width"] * wl["height"] * 3
    first = [sc.render_view(v, 0, 8) for v in range(nv)]
    st = pb.initialize(cfg, first)
    P = st.canvas_width * st.canvas_height
    pin_in = [lib.stitch_b200_host_alloc(fb) for _ in range(nv)]
    pg_in = [np.ascontiguousarray(first[v].data).reshape(-1).copy() for v in range(nv)]
    for v in range(nv):
        C.memmove(pin_in[v], pg_in[v].ctypes.data, fb)
    pin_ptrs = (C.c_void_p * nv)(*pin_in)
    pg_ptrs = (C.c_void_p * nv)(*[a.ctypes.data for a in pg_in])
    pin_out = (lib.stitch_b200_host_alloc(P * 3), lib.stitch_b200_host_alloc(P))
    pg_out = (np.zeros(P * 3, np.uint8), np.zeros(P, np.uint8))
    pg_out_p = (pg_out[0].ctypes.data, pg_out[1].ctypes.data)
    res = {}

    def timeit(name, ins, outs):
        for _ in range(3):
            pb.pipeline.check(lib.stitch_b200_process(st.handle, ins, outs[0], outs[1], None))
        t = time.perf_counter()
        for _ in range(reps):
            pb.pipeline.check(lib.stitch_b200_process(st.handle, ins, outs[0], outs[1], None))
        res[name] = round((time.perf_counter() - t) / reps * 1e3, 3)

    for _ in range(2):
        timeit("pinned_in_pinned_out_ms", pin_ptrs, pin_out)
        timeit("pageable_in_pinned_out_ms", pg_ptrs, pin_out)
        timeit("pinned_in_pageable_out_ms", pin_ptrs, pg_out_p)
        timeit("pageable_in_pageable_out_ms", pg_ptrs, pg_out_p)
    a = np.ones(P * 4, np.uint8)
    b = np.zeros_like(a)
    np.copyto(b, a)
    t = time.perf_counter()
    for _ in range(10):
        np.copyto(b, a)
    res["numpy_memcpy_gbs_1thread"] = round(10 * a.nbytes / (time.perf_counter() - t) / 1e9, 1)
    res["copy_threads_env"] = os.environ.get("STITCH_B200_COPY_THREADS", "default")
    res["host_cores"] = os.cpu_count()
    print(json.dumps(res))
    st.close()


if __name__ == "__main__":
    main()
