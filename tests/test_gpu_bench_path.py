"""Parity of the path bench.py times (BASELINE configs[1], C2: 4 x 1920x1080,
300 frames): stitch_b200_process_device_async with four frames in flight over
the context's pipeline slots inside one fork/join -- exactly the bench's
`value` loop, frame sets cycling over the same 16 pre-rendered inputs --
against the synchronous C-ABI call (stitch_b200_process) on a second context
and against the CPU oracle, every 10th panorama (RGB + mask) compared
bit-for-bit over all 300 frames, so the temporal state the four slots chain
(3D-M windows, threshold history) is exercised for the whole sequence."""
import ctypes as C
import os

import numpy as np
import pytest

import bench
import paper_2308_09209_b200 as pb
from paper_2308_09209_b200 import _abi

FRAMES = int(os.environ.get("STITCH_B200_BENCH_PATH_FRAMES", "300"))
SETS = 16
EVERY = 10


@pytest.mark.gpu
def test_bench_async_path_300_frames_matches_sync_and_oracle():
    lib = _abi.load()
    wl = bench.WORKLOADS["c2"]
    threads = bench.cpu_cores()
    sc = bench.build_scene(wl, seed=1)
    nv = wl["views"]
    fb = wl["width"] * wl["height"] * 3
    sets = [[sc.render_view(v, t, threads) for v in range(nv)] for t in range(SETS)]
    dev, host = [], []
    for t in range(SETS):
        ds, hs = [], []
        for v in range(nv):
            hp = lib.stitch_b200_host_alloc(fb)
            C.memmove(hp, np.ascontiguousarray(sets[t][v].data).ctypes.data, fb)
            dp = lib.stitch_b200_device_alloc(0, fb)
            pb.pipeline.check(lib.stitch_b200_memcpy_h2d(dp, hp, fb))
            ds.append(dp)
            hs.append(hp)
        dev.append((C.c_void_p * nv)(*ds))
        host.append((C.c_void_p * nv)(*hs))
    cfg = sc.config()  # refinement on, as bench.py
    a = pb.initialize(cfg, sets[0])
    b = pb.initialize(cfg, sets[0])
    ref = bench.CpuRunner(wl, "port", threads)  # the oracle, refined on the same first frames
    w, h = a.canvas_width, a.canvas_height
    assert (w, h) == (b.canvas_width, b.canvas_height)
    n = w * h
    sync_rgb = lib.stitch_b200_host_alloc(n * 3)
    sync_mask = lib.stitch_b200_host_alloc(n)
    got_rgb = np.empty((h, w, 3), np.uint8)
    got_mask = np.empty((h, w), np.uint8)
    prgb, pmask = C.c_void_p(), C.c_void_p()
    checked = 0
    try:
        pb.pipeline.check(lib.stitch_b200_fork(a.handle))
        for i in range(FRAMES):
            pb.pipeline.check(lib.stitch_b200_process_device_async(a.handle, dev[i % SETS]))
            pb.pipeline.check(lib.stitch_b200_process(b.handle, host[i % SETS], sync_rgb,
                                                      sync_mask, None))
            odata, omask, _ = ref.st.process([s.data for s in sets[i % SETS]])
            if i % EVERY != EVERY - 1 and i != FRAMES - 1:
                continue
            # frame i's outputs live until frame i + 4 is enqueued: join, read, fork
            pb.pipeline.check(lib.stitch_b200_join(a.handle))
            pb.pipeline.check(lib.stitch_b200_synchronize(a.handle))
            pb.pipeline.check(lib.stitch_b200_device_pano(a.handle, C.byref(prgb), C.byref(pmask)))
            pb.pipeline.check(lib.stitch_b200_memcpy_d2h(got_rgb.ctypes.data, prgb, n * 3))
            pb.pipeline.check(lib.stitch_b200_memcpy_d2h(got_mask.ctypes.data, pmask, n))
            pb.pipeline.check(lib.stitch_b200_fork(a.handle))
            srgb = np.ctypeslib.as_array(C.cast(sync_rgb, C.POINTER(C.c_uint8)), (n * 3,))
            smask = np.ctypeslib.as_array(C.cast(sync_mask, C.POINTER(C.c_uint8)), (n,))
            assert np.array_equal(got_mask, smask.reshape(h, w)), f"frame {i}: async mask != sync"
            assert np.array_equal(got_rgb, srgb.reshape(h, w, 3)), f"frame {i}: async rgb != sync"
            assert np.array_equal(got_mask, omask), f"frame {i}: mask != oracle"
            d = int(np.abs(got_rgb.astype(np.int16) - odata.astype(np.int16)).max())
            assert d == 0, f"frame {i}: panorama differs from the oracle by {d} LSB"
            checked += 1
        pb.pipeline.check(lib.stitch_b200_join(a.handle))
        pb.pipeline.check(lib.stitch_b200_synchronize(a.handle))
        assert checked == sum(1 for i in range(FRAMES) if i % EVERY == EVERY - 1 or i == FRAMES - 1)
    finally:
        ref.close()
        a.close()
        b.close()
        for t in range(SETS):
            for v in range(nv):
                lib.stitch_b200_host_free(host[t][v])
                lib.stitch_b200_device_free(dev[t][v])
        lib.stitch_b200_host_free(sync_rgb)
        lib.stitch_b200_host_free(sync_mask)
