"""Interleaved A/B of the synchronous call's pageable input staging modes
(STITCH_B200_STAGE_MODE / _CHUNK_MB, read per call) at C2; median ms per call."""
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
    lib = _abi.load()
    wl = bench.WORKLOADS["c2"]
    sc = bench.build_scene(wl, seed=1)
    nv = wl["views"]
    fb = wl["width"] * wl["height"] * 3
    first = [sc.render_view(v, 0, 8) for v in range(nv)]
    st = pb.initialize(sc.config(), first)
    P = st.canvas_width * st.canvas_height
    pg_in = [np.ascontiguousarray(first[v].data).reshape(-1).copy() for v in range(nv)]
    pg_ptrs = (C.c_void_p * nv)(*[a.ctypes.data for a in pg_in])
    pin_out = (lib.stitch_b200_host_alloc(P * 3), lib.stitch_b200_host_alloc(P))
    pg_out = (np.zeros(P * 3, np.uint8), np.zeros(P, np.uint8))
    outs = {"pin_out": pin_out, "pg_out": (pg_out[0].ctypes.data, pg_out[1].ctypes.data)}
    cfgs = [(m, c) for m, c in ((0, 4), (1, 4), (2, 1), (2, 2), (2, 4), (2, 8))]
    samples = {}
    for rnd in range(6):
        for m, c in cfgs:
            os.environ["STITCH_B200_STAGE_MODE"] = str(m)
            os.environ["STITCH_B200_STAGE_CHUNK_MB"] = str(c)
            for on, o in outs.items():
                for _ in range(2):
                    pb.pipeline.check(lib.stitch_b200_process(st.handle, pg_ptrs, o[0], o[1], None))
                ts = []
                for _ in range(15):
                    t = time.perf_counter()
                    pb.pipeline.check(lib.stitch_b200_process(st.handle, pg_ptrs, o[0], o[1], None))
                    ts.append(time.perf_counter() - t)
                samples.setdefault(f"m{m}_c{c}_{on}", []).extend(ts)
    res = {k: round(float(np.median(v)) * 1e3, 3) for k, v in samples.items()}
    res["threads"] = os.environ.get("STITCH_B200_COPY_THREADS", "default")
    print(json.dumps(res))
    st.close()


if __name__ == "__main__":
    main()
