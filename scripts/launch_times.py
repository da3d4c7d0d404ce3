"""Per-launch device times of one frame (eager plan, CUDA events around each
launch) for the bench workload; prints kind, milliseconds."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2308_09209_b200 as pb  # noqa: E402
from paper_2308_09209_b200 import _abi  # noqa: E402

lib = _abi.load()
wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
sc = bench.build_scene(wl, 1)
cfg = sc.config()
nv = wl["views"]
fb = wl["width"] * wl["height"] * 3
ptrs = []
for v in range(nv):
    img = sc.render_view(v, 0, 16).data
    dp = lib.stitch_b200_device_alloc(0, fb)
    pb.pipeline.check(lib.stitch_b200_memcpy_h2d(dp, img.ctypes.data, fb))
    ptrs.append(dp)
dev = (C.c_void_p * nv)(*ptrs)
state = pb.initialize(cfg, [pb.Frame(np.zeros((wl["height"], wl["width"], 3), np.uint8))] * nv)
kinds = (C.c_int * 512)()
ms = (C.c_float * 512)()
for it in range(4):
    n = lib.stitch_b200_profile_frame(state.handle, dev, 512, kinds, ms)
tot = 0.0
for i in range(n):
    print(f"{i:3d} {_abi.OP_KIND_NAMES[kinds[i]]:14s} {ms[i]*1e3:9.1f} us")
    tot += ms[i]
print(f"total {tot:.4f} ms")
