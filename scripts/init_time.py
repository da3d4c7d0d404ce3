import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np
import bench
import paper_2308_09209_b200 as pb
for key in ("c2", "c3", "c4"):
    wl = bench.WORKLOADS[key]
    sc = bench.build_scene(wl, 1)
    cfg = sc.config()
    fr = [pb.Frame(np.zeros((wl["height"], wl["width"], 3), np.uint8))] * wl["views"]
    st = pb.initialize(cfg, fr); st.close() if hasattr(st, "close") else None
    t0 = time.perf_counter()
    st = pb.initialize(cfg, fr)
    t1 = time.perf_counter()
    print(key, "initialize s", round(t1 - t0, 3))
