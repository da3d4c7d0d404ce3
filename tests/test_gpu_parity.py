"""GPU parity: the B200 path (through the C ABI) against the CPU oracle on
identical synthetic inputs.

Contract (BASELINE.json north_star): warp/flow fields within 1e-3 px, colour
matrices within 1e-4 relative, final 8-bit panoramas within +-1 LSB with an
identical mask.  The implementation is designed to be bit-exact (FP64 warp,
integer-exact colour moments, FP32 flow with --fmad=false), so these tests
assert the tolerance AND report the max-abs-diff; the bit-exact expectation
is asserted separately where the arithmetic is integer/byte work.
"""
import ctypes as C

import numpy as np
import pytest

import oracle as O
import paper_2308_09209_b200 as pb
from paper_2308_09209_b200 import _abi
from tests.helpers import frames_at, maxdiff, oracle_config, product_config, scene

pytestmark = pytest.mark.gpu

M_RTOL = 1e-4
FLOW_TOL = 1e-3


def _lib():
    return _abi.load()


def make_pair(sc, frames0=None, **kw):
    cfg = product_config(sc, **kw)
    first = frames0 or frames_at(sc, 0)
    state = pb.initialize(cfg, first)
    ost = O.OracleState(oracle_config(sc, **kw))
    return state, ost


def debug_flow(state, k, d, shape):
    u = np.zeros(shape, np.float32)
    v = np.zeros(shape, np.float32)
    pb.pipeline.check(_lib().stitch_b200_debug_flow(state.handle, k, d,
                                                    u.ctypes.data_as(C.c_void_p),
                                                    v.ctypes.data_as(C.c_void_p)))
    return u, v


def debug_warp(state, view, frame):
    w, h = state.canvas_width, state.canvas_height
    rgb = np.zeros((h, w, 3), np.uint8)
    mask = np.zeros((h, w), np.uint8)
    src = np.ascontiguousarray(frame.data)
    pb.pipeline.check(_lib().stitch_b200_debug_warp_view(state.handle, view,
                                                         src.ctypes.data_as(C.c_void_p),
                                                         rgb.ctypes.data_as(C.c_void_p),
                                                         mask.ctypes.data_as(C.c_void_p)))
    return rgb, mask


def check_geometry(state, ost, n_views):
    assert state.canvas == ost.canvas
    assert len(state.pairs) == ost.n_pairs()
    for v in range(n_views):
        _, inv = ost.maps(v)
        np.testing.assert_array_equal(state.inv_map(v), inv)
        assert state.view_bbox(v) == ost.view_bbox(v)
    for k, p in enumerate(state.pairs):
        view, partner, bounds = ost.pair(k)
        assert (p.view, p.partner, p.bounds) == (view, partner, bounds)
        np.testing.assert_array_equal(p.theta_i, ost.pair_weights(k))


def check_frame(state, ost, frames, t, *, exact=True):
    res = pb.process_frame(state, frames)
    odata, omask, orep = ost.process([f.data for f in frames])
    rep = res.report
    # colour matrices (1e-4 relative; bit-exact expected)
    for k in range(len(state.pairs)):
        m_ref = np.array(orep.m[k][:]).reshape(3, 3)
        m = rep.color_matrices[k]
        np.testing.assert_allclose(m, m_ref, rtol=M_RTOL, atol=1e-12)
        if exact:
            np.testing.assert_array_equal(m, m_ref)
        assert rep.rank_deficient[k] == bool(orep.rank_deficient[k])
    # flows (1e-3 px; bit-exact expected)
    for k, p in enumerate(state.pairs):
        shape = (p.bounds[3] - p.bounds[1], p.bounds[2] - p.bounds[0])
        for d in range(2):
            u, v = debug_flow(state, k, d, shape)
            ou, ov = ost.last_flow(k, d)
            assert np.abs(u - ou).max() <= FLOW_TOL, (t, k, d, np.abs(u - ou).max())
            assert np.abs(v - ov).max() <= FLOW_TOL
            if exact:
                np.testing.assert_array_equal(u, ou)
                np.testing.assert_array_equal(v, ov)
    # balancing thresholds
    assert rep.balanced == bool(orep.balanced)
    assert rep.threshold_m1 == list(orep.threshold_m1)
    assert rep.threshold_m2 == list(orep.threshold_m2)
    assert rep.frame_index == orep.frame_index
    # panorama: identical mask, +-1 LSB (bit-exact expected)
    np.testing.assert_array_equal(res.panorama.mask, omask)
    d = maxdiff(res.panorama.data, odata)
    assert d <= 1, f"frame {t}: max abs diff {d}"
    if exact:
        assert d == 0, f"frame {t}: max abs diff {d}"
    return res


@pytest.mark.parametrize("views", [2, 3])
def test_init_geometry_matches_oracle(views):
    sc = scene(views=views, width=200, height=150)
    state, ost = make_pair(sc)
    check_geometry(state, ost, views)


def test_warp_views_bit_exact():
    sc = scene(views=3, width=160, height=120)
    state, ost = make_pair(sc)
    frames = frames_at(sc, 0)
    ost.process([f.data for f in frames])
    for v in range(3):
        rgb, mask = debug_warp(state, v, frames[v])
        orgb, omask = ost.last_warped(v)
        np.testing.assert_array_equal(mask, omask)
        np.testing.assert_array_equal(rgb, orgb)


def test_c1_config_parity_all_stages():
    """BASELINE config 1: 2 x 640x480, one overlap, fixed homography; casts,
    a flicker event and a moving parallax object; several frames so the
    3-frame windows fill and roll."""
    sc = scene(views=2, width=640, height=480, frames=6, casts=[(1, 1, 1), (0.85, 1.0, 1.1)],
               flicker=[pb.FlickerEvent(frame=3, view=1, gains=(1.2, 1.1, 0.9))])
    state, ost = make_pair(sc)
    check_geometry(state, ost, 2)
    for t in range(6):
        check_frame(state, ost, frames_at(sc, t), t)


@pytest.mark.parametrize("kw", [dict(), dict(window=1), dict(weighting=1), dict(window=2),
                                dict(levels=2, iterations=20)])
def test_three_view_parity(kw):
    sc = scene(views=3, width=200, height=150, frames=4, casts=[(0.9, 1, 1), (1, 1, 1),
                                                                (1, 0.95, 1.1)])
    state, ost = make_pair(sc, **kw)
    check_geometry(state, ost, 3)
    for t in range(4):
        check_frame(state, ost, frames_at(sc, t), t)


def test_four_view_chain_parity():
    """N-view extension (chain topology, strip rig): parity vs the extended
    oracle (unpinned by the reference, which caps views at 3)."""
    sc = scene(views=4, width=200, height=150, frames=3, focal_scale=1.03,
               casts=[(0.9, 1, 1), (1, 1, 1), (1, 0.95, 1.1), (1.1, 1, 0.9)])
    state, ost = make_pair(sc)
    check_geometry(state, ost, 4)
    for t in range(3):
        check_frame(state, ost, frames_at(sc, t), t)


def test_tiny_overlap_degrades_to_zero_flow():
    # overlap shorter than 16 rows -> dense_flow throws TooSmall -> zero flow
    sc = scene(views=2, width=160, height=14, obj=False)
    state, ost = make_pair(sc)
    p = state.pairs[0]
    assert p.bounds[2] - p.bounds[0] < 16 or p.bounds[3] - p.bounds[1] < 16
    for t in range(2):
        check_frame(state, ost, frames_at(sc, t), t)


def test_flat_overlap_rank_deficient_identity():
    # a constant scene makes X^T X rank one -> RankDeficient -> identity M
    sc = scene(views=2, width=120, height=90, obj=False)
    frames = [pb.Frame(np.full_like(f.data, 77)) for f in frames_at(sc, 0)]
    state, ost = make_pair(sc, frames0=frames)
    res = check_frame(state, ost, frames, 0)
    assert res.report.rank_deficient == [True]
    np.testing.assert_array_equal(res.report.color_matrices[0], np.eye(3))


def test_run_sequence_and_determinism():
    sc = scene(views=2, width=160, height=120, frames=3)
    cfg = product_config(sc)
    streams = sc.render_streams()
    a = pb.run_sequence(cfg, streams)
    b = pb.run_sequence(cfg, streams)
    assert a.report.frames == 3 and len(a.panoramas) == 3
    for x, y in zip(a.panoramas, b.panoramas):
        np.testing.assert_array_equal(x.data, y.data)
        np.testing.assert_array_equal(x.mask, y.mask)
    assert all(t >= 0 for t in a.report.totals)


def test_errors_fail_loudly():
    sc = scene(views=2, width=120, height=90)
    cfg = product_config(sc)
    cfg.refine.enabled = True
    cfg.projection = "cylindrical"  # refinement serves the planar canvas only
    with pytest.raises(pb.StitchError):
        pb.initialize(cfg, frames_at(sc, 0))
    cfg = product_config(sc, lam=0.7)
    with pytest.raises(pb.StitchError) as e:
        pb.initialize(cfg, frames_at(sc, 0))
    assert e.value.code == pb.ErrorCode.ConfigError
    cfg = product_config(sc)
    state = pb.initialize(cfg, frames_at(sc, 0))
    with pytest.raises(pb.StitchError):
        pb.process_frame(state, frames_at(sc, 0)[:1])


def test_update_geometry_keeps_temporal_state():
    """Re-refinement (pipeline.cpp:395-406) keeps windows, history, counter."""
    sc = scene(views=2, width=160, height=120, frames=4, casts=[(1, 1, 1), (0.8, 1, 1.1)])
    state, ost = make_pair(sc)
    for t in range(2):
        check_frame(state, ost, frames_at(sc, t), t)
    # re-upload the same geometry through the drop-in snapshot path
    init = _abi.Init()
    w, h, ox, oy = state.canvas
    init.canvas_width, init.canvas_height = w, h
    init.canvas_offset[0], init.canvas_offset[1] = ox, oy
    init.n_views, init.reference = 2, sc.reference_view()
    keep = []
    for v in range(2):
        init.view_width[v], init.view_height[v] = 160, 120
        inv = state.inv_map(v).reshape(9)
        for i in range(9):
            init.inv_maps[v][i] = inv[i]
    init.n_pairs = len(state.pairs)
    for k, p in enumerate(state.pairs):
        th = np.ascontiguousarray(p.theta_i, np.float32)
        keep.append(th)
        init.pairs[k].view, init.pairs[k].partner = p.view, p.partner
        init.pairs[k].x0, init.pairs[k].y0, init.pairs[k].x1, init.pairs[k].y1 = p.bounds
        init.pairs[k].theta_i = th.ctypes.data_as(C.POINTER(C.c_float))
    init.window_capacity = 3
    init.lambda_, init.gamma_dark, init.gamma_bright = 0.05, 1.5, 1.5
    init.target_black, init.target_white = 0, 255
    init.flow_levels, init.flow_iterations, init.smoothness = 4, 50, 15.0
    init.fuse_weighting = 0
    pb.pipeline.check(_lib().stitch_b200_update_geometry(state.handle, C.byref(init)))
    for t in range(2, 4):
        check_frame(state, ost, frames_at(sc, t), t)


def test_update_maps_rebuilds_geometry_on_device():
    """Re-refinement from new homographies (stitch_b200_update_maps): the
    canvas, inverse maps and device-built pair geometry equal a fresh
    initialize() with those maps, and the temporal state is carried over."""
    sc1 = scene(views=3, width=160, height=120, frames=4, focal_scale=1.0)
    sc2 = scene(views=3, width=160, height=120, frames=4, focal_scale=1.03)
    cfg1, cfg2 = product_config(sc1), product_config(sc2)
    state = pb.initialize(cfg1, frames_at(sc1, 0))
    for t in range(2):
        pb.process_frame(state, frames_at(sc1, t))
    sizes = [(160, 120)] * 3
    maps2 = pb.camera_maps(cfg2, sizes)
    assert not np.array_equal(maps2, pb.camera_maps(cfg1, sizes))
    state.update_maps(maps2)
    fresh = pb.initialize(cfg2, frames_at(sc2, 0))
    assert state.canvas == fresh.canvas
    for v in range(3):
        assert np.array_equal(state.inv_map(v), fresh.inv_map(v))
        assert state.view_bbox(v) == fresh.view_bbox(v)
    assert len(state.pairs) == len(fresh.pairs)
    for a, b in zip(state.pairs, fresh.pairs):
        assert (a.view, a.partner, a.bounds) == (b.view, b.partner, b.bounds)
        assert np.array_equal(a.theta_i, b.theta_i)
    r1 = pb.process_frame(state, frames_at(sc2, 2))
    r2 = pb.process_frame(fresh, frames_at(sc2, 2))
    assert r1.report.frame_index == 2 and r2.report.frame_index == 0
    assert r1.panorama.data.shape == r2.panorama.data.shape
    # the unchanged maps reproduce the initialize() geometry bit for bit
    state.update_maps(pb.camera_maps(cfg1, sizes))
    again = pb.initialize(cfg1, frames_at(sc1, 0))
    for a, b in zip(state.pairs, again.pairs):
        assert a.bounds == b.bounds and np.array_equal(a.theta_i, b.theta_i)
    state.close()
    fresh.close()
    again.close()


def test_create_from_snapshot_matches_initialize():
    sc = scene(views=2, width=160, height=120, frames=2)
    state, ost = make_pair(sc)
    init = _abi.Init()
    w, h, ox, oy = state.canvas
    init.canvas_width, init.canvas_height = w, h
    init.canvas_offset[0], init.canvas_offset[1] = ox, oy
    init.n_views, init.reference = 2, sc.reference_view()
    for v in range(2):
        init.view_width[v], init.view_height[v] = 160, 120
        inv = state.inv_map(v).reshape(9)
        for i in range(9):
            init.inv_maps[v][i] = inv[i]
    init.n_pairs = 1
    p = state.pairs[0]
    th = np.ascontiguousarray(p.theta_i, np.float32)
    init.pairs[0].view, init.pairs[0].partner = p.view, p.partner
    init.pairs[0].x0, init.pairs[0].y0, init.pairs[0].x1, init.pairs[0].y1 = p.bounds
    init.pairs[0].theta_i = th.ctypes.data_as(C.POINTER(C.c_float))
    init.window_capacity = 3
    init.lambda_, init.gamma_dark, init.gamma_bright = 0.05, 1.5, 1.5
    init.target_black, init.target_white = 0, 255
    init.flow_levels, init.flow_iterations, init.smoothness = 4, 50, 15.0
    snap = pb.create_from_init(init, 0, product_config(sc))
    for t in range(2):
        fr = frames_at(sc, t)
        a = pb.process_frame(state, fr)
        b = pb.process_frame(snap, fr)
        np.testing.assert_array_equal(a.panorama.data, b.panorama.data)


@pytest.mark.parametrize("env", [{"STITCH_B200_HS_FORCE_EXACT": "1"},
                                 {"STITCH_B200_HS_VARIANT": "0"},
                                 {"STITCH_B200_HS_VARIANT": "1"},
                                 {"STITCH_B200_HS_VARIANT": "5"},
                                 {"STITCH_B200_HS_VARIANT": "5",
                                  "STITCH_B200_HS_FORCE_EXACT": "1"},
                                 {"STITCH_B200_HS_SEGS": "1"},
                                 {"STITCH_B200_HS_SEGS": "3"},
                                 {"STITCH_B200_HS_SEGS": "10", "STITCH_B200_HS_VARIANT": "5"},
                                 {"STITCH_B200_PREP_VARIANT": "0", "STITCH_B200_HS_FUSE": "0"},
                                 {"STITCH_B200_HS_FUSE": "0"},
                                 {"STITCH_B200_HS_XL": "1"},
                                 {"STITCH_B200_HS_ELIN": "0"},
                                 {"STITCH_B200_HS_VARIANT": "6", "STITCH_B200_HS_ELIN_TALL": "1"},
                                 {"STITCH_B200_HS_SEGS": "1", "STITCH_B200_HS_FUSE": "0"},
                                 {"STITCH_B200_HS_VARIANT": "7"},
                                 {"STITCH_B200_HS_VARIANT": "6", "STITCH_B200_HS_FORCE_EXACT": "1"},
                                 {"STITCH_B200_CANVAS_CLASS": "0"},
                                 {"STITCH_B200_HS_TALL_MIN": "1"},
                                 {"STITCH_B200_HS_TALL_MIN": "1", "STITCH_B200_HS_ELIN_TALL": "2"},
                                 {"STITCH_B200_HS_SPLIT": "0"},
                                 {"STITCH_B200_PYR_FUSE": "0"},
                                 {"STITCH_B200_WARP_STAGE": "1"},
                                 {"STITCH_B200_COLOR_VEC": "0", "STITCH_B200_COLOR_SPLIT": "0"},
                                 {"STITCH_B200_COLOR_VEC": "1", "STITCH_B200_COLOR_SPLIT": "0"},
                                 {"STITCH_B200_CANVAS_SPLIT": "0"},
                                 {"STITCH_B200_HS_TMA": "1"},
                                 {"STITCH_B200_PDL": "0"},
                                 {"STITCH_B200_PDL": "2"},
                                 {"STITCH_B200_HS_PAIR": "1"},
                                 {"STITCH_B200_HS_PAIR": "1", "STITCH_B200_HS_FORCE_EXACT": "1"}])
def test_flow_kernel_variants_bit_exact(env):
    """The register-blocked Jacobi kernel's region variants, sweep
    segmentations and its exact IEEE-division fallback path (forced) all
    reproduce the oracle's flows; run in a subprocess because the switches
    are read once per process."""
    import os
    import subprocess
    import sys

    code = ("import tests.test_gpu_parity as T; T.test_c1_config_parity_all_stages(); "
            "T.test_three_view_parity({})")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env={**os.environ, **env},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def test_pipelined_submit_matches_sync_and_oracle():
    """stitch_b200_submit/wait (two frames in flight, pinned host buffers)
    produces exactly the synchronous path's panoramas and reports."""
    sc = scene(views=3, width=200, height=150, frames=5,
               casts=[(0.9, 1, 1), (1, 1, 1), (1, 0.95, 1.1)])
    state, ost = make_pair(sc)
    lib = _lib()
    w, h = state.canvas_width, state.canvas_height
    n = w * h
    nv = 3
    fb = 200 * 150 * 3
    hin = [[lib.stitch_b200_host_alloc(fb) for _ in range(nv)] for _ in range(5)]
    hout = [(lib.stitch_b200_host_alloc(n * 3), lib.stitch_b200_host_alloc(n)) for _ in range(5)]
    try:
        tickets = []
        reps = []
        for t in range(5):
            for v, f in enumerate(frames_at(sc, t)):
                C.memmove(hin[t][v], np.ascontiguousarray(f.data).ctypes.data, fb)
            tk = C.c_longlong()
            pb.pipeline.check(lib.stitch_b200_submit(state.handle, (C.c_void_p * nv)(*hin[t]),
                                                     hout[t][0], hout[t][1], C.byref(tk)))
            tickets.append(tk.value)
            if t >= 1:
                r = _abi.Report()
                pb.pipeline.check(lib.stitch_b200_wait(state.handle, tickets[t - 1], C.byref(r)))
                reps.append(r)
        r = _abi.Report()
        pb.pipeline.check(lib.stitch_b200_wait(state.handle, tickets[-1], C.byref(r)))
        reps.append(r)
        for t in range(5):
            odata, omask, orep = ost.process([f.data for f in frames_at(sc, t)])
            rgb = np.ctypeslib.as_array(C.cast(hout[t][0], C.POINTER(C.c_uint8)), (n * 3,))
            msk = np.ctypeslib.as_array(C.cast(hout[t][1], C.POINTER(C.c_uint8)), (n,))
            np.testing.assert_array_equal(rgb.reshape(h, w, 3), odata)
            np.testing.assert_array_equal(msk.reshape(h, w), omask)
            assert reps[t].frame_index == t
            for k in range(2):
                np.testing.assert_array_equal(np.array(reps[t].color_matrices[k][:]),
                                              np.array(orep.m[k][:]))
    finally:
        for t in range(5):
            for p in hin[t]:
                lib.stitch_b200_host_free(p)
            lib.stitch_b200_host_free(hout[t][0])
            lib.stitch_b200_host_free(hout[t][1])


def test_eight_view_chain_parity():
    """Config-4 topology (8 cameras, chain of 7 pairs, depth 4 colour
    correction) at reduced resolution, bit-exact vs the extended oracle."""
    casts = [(1.0 - 0.03 * v, 1.0, 1.0 + 0.02 * v) for v in range(8)]
    sc = scene(views=8, width=240, height=135, frames=2, focal_scale=1.03, casts=casts)
    state, ost = make_pair(sc)
    check_geometry(state, ost, 8)
    assert len(state.pairs) == 7
    for t in range(2):
        check_frame(state, ost, frames_at(sc, t), t)


def test_sixteen_view_chain_parity():
    """The maximum view count (STITCH_B200_MAX_VIEWS = 16, 15 chain pairs,
    colour-correction depth 8) at small frames, bit-exact vs the oracle."""
    casts = [(1.0 - 0.02 * v, 1.0, 1.0 + 0.015 * v) for v in range(16)]
    sc = scene(views=16, width=128, height=96, frames=2, focal_scale=1.02, casts=casts)
    state, ost = make_pair(sc)
    check_geometry(state, ost, 16)
    assert len(state.pairs) == 15
    for t in range(2):
        check_frame(state, ost, frames_at(sc, t), t)


def test_ring_360_parity():
    """BASELINE config 3 topology: 6-camera 360-degree ring on a cylindrical
    canvas (extension: lift tables, ring-chain pairs, the opposite view
    straddling the seam), bit-exact vs the extended oracle."""
    spec = pb.SynthSpec(views=6, width=256, height=144, frames=3, rig="ring",
                        color_casts=[(1.0 - 0.04 * v, 1.0, 1.0 + 0.03 * v) for v in range(6)])
    sc = pb.SynthScene(spec)
    state, ost = make_pair(sc)
    check_geometry(state, ost, 6)
    assert [(p.view, p.partner) for p in state.pairs] == [(1, 0), (5, 0), (2, 1), (4, 5), (3, 2)]
    for t in range(3):
        check_frame(state, ost, frames_at(sc, t), t)


def test_heterogeneous_camera_sizes():
    """Views of different sizes (the reference's Frame sizes are per view):
    view 2's frames are a cropped window of the synthetic camera, with the
    principal point shifted accordingly (a cropped pinhole image)."""
    sc = scene(views=3, width=240, height=180, frames=3,
               casts=[(1, 1, 1), (0.9, 1.0, 1.1), (1.1, 0.95, 1.0)])
    cfg = product_config(sc)
    x0, y0, cw, ch = 24, 12, 200, 150
    cfg.views[2].intrinsics.cx -= x0
    cfg.views[2].intrinsics.cy -= y0

    def frames(t):
        fs = frames_at(sc, t)
        fs[2] = pb.Frame(np.ascontiguousarray(fs[2].data[y0:y0 + ch, x0:x0 + cw]))
        return fs

    state = pb.initialize(cfg, frames(0))
    cams = []
    for v in cfg.views:
        r = np.asarray(v.extrinsics.rotation, np.float64).reshape(9)
        t = np.asarray(v.extrinsics.translation, np.float64).reshape(3)
        cams.append((v.intrinsics.fx, v.intrinsics.fy, v.intrinsics.cx, v.intrinsics.cy,
                     list(r), list(t)))
    sizes = [(240, 180), (240, 180), (cw, ch)]
    ost = O.OracleState(O.make_config(3, cfg.reference, sizes, cams, threads=4, keep_debug=1))
    check_geometry(state, ost, 3)
    for t in range(3):
        check_frame(state, ost, frames(t), t)
    state.close()


def test_concurrent_contexts_on_host_threads():
    """Two panorama streams on their own contexts, driven from two host
    threads at once (ctypes releases the GIL in the C ABI calls): each
    stream's panoramas and reports equal its own sequential run."""
    import threading

    scs = [scene(views=3, width=200, height=150, frames=4, seed=s,
                 casts=[(0.9, 1, 1), (1, 1, 1), (1, 0.95, 1.1)]) for s in (3, 4)]
    expect = []
    for sc in scs:
        st = pb.initialize(product_config(sc), frames_at(sc, 0))
        expect.append([pb.process_frame(st, frames_at(sc, t)) for t in range(4)])
        st.close()
    got = [None, None]
    errs = []

    def run(i):
        try:
            sc = scs[i]
            st = pb.initialize(product_config(sc), frames_at(sc, 0))
            got[i] = [pb.process_frame(st, frames_at(sc, t)) for t in range(4)]
            st.close()
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for i in range(2):
        for t in range(4):
            np.testing.assert_array_equal(got[i][t].panorama.data, expect[i][t].panorama.data)
            np.testing.assert_array_equal(got[i][t].panorama.mask, expect[i][t].panorama.mask)
            np.testing.assert_array_equal(np.array(got[i][t].report.color_matrices),
                                          np.array(expect[i][t].report.color_matrices))


def test_tickets_survive_geometry_update():
    """Host-path frames still in flight when the geometry is replaced
    (stitch_b200_update_maps -> a fresh context) keep their reports, and ticket
    numbers stay monotonic across the swap, so an old ticket never aliases a
    new frame."""
    sc = scene(views=2, width=160, height=120, frames=4)
    cfg = product_config(sc)
    state = pb.initialize(cfg, frames_at(sc, 0))
    lib = _lib()
    w, h = state.canvas_width, state.canvas_height
    fb = 160 * 120 * 3
    hin = [[lib.stitch_b200_host_alloc(fb) for _ in range(2)] for _ in range(3)]
    hout = [(lib.stitch_b200_host_alloc(w * h * 3), lib.stitch_b200_host_alloc(w * h))
            for _ in range(3)]
    try:
        tickets = []
        for t in range(3):
            for v, f in enumerate(frames_at(sc, t)):
                C.memmove(hin[t][v], np.ascontiguousarray(f.data).ctypes.data, fb)
        for t in range(2):
            tk = C.c_longlong()
            pb.pipeline.check(lib.stitch_b200_submit(state.handle, (C.c_void_p * 2)(*hin[t]),
                                                     hout[t][0], hout[t][1], C.byref(tk)))
            tickets.append(tk.value)
        state.update_maps(pb.camera_maps(cfg, [(160, 120)] * 2))
        tk = C.c_longlong()
        pb.pipeline.check(lib.stitch_b200_submit(state.handle, (C.c_void_p * 2)(*hin[2]),
                                                 hout[2][0], hout[2][1], C.byref(tk)))
        tickets.append(tk.value)
        assert tickets == sorted(set(tickets))
        for t, tk in enumerate(tickets):
            r = _abi.Report()
            pb.pipeline.check(lib.stitch_b200_wait(state.handle, tk, C.byref(r)))
            assert r.frame_index == t
    finally:
        state.close()
        for t in range(3):
            for p in hin[t]:
                lib.stitch_b200_host_free(p)
            lib.stitch_b200_host_free(hout[t][0])
            lib.stitch_b200_host_free(hout[t][1])


def test_pageable_submit_matches_pinned():
    """The reference's caller passes pageable std::vector buffers: submit/wait
    with pageable (numpy) frames and outputs, four frames in flight, goes
    through the context's pinned staging ring and yields exactly the pinned
    path's panoramas and reports."""
    sc = scene(views=3, width=200, height=150, frames=7,
               casts=[(0.9, 1, 1), (1, 1, 1), (1, 0.95, 1.1)])
    lib = _lib()
    cfg = product_config(sc)
    a = pb.initialize(cfg, frames_at(sc, 0))
    w, h = a.canvas_width, a.canvas_height
    try:
        want = [pb.process_frame(a, frames_at(sc, t)) for t in range(7)]  # sync path
    finally:
        a.close()
    b = pb.initialize(cfg, frames_at(sc, 0))
    ins = [[np.ascontiguousarray(f.data) for f in frames_at(sc, t)] for t in range(7)]
    outs = [(np.zeros((h, w, 3), np.uint8), np.zeros((h, w), np.uint8)) for _ in range(7)]
    try:
        tickets, reps = [], {}
        for t in range(7):
            tk = C.c_longlong()
            pb.pipeline.check(lib.stitch_b200_submit(
                b.handle, (C.c_void_p * 3)(*[x.ctypes.data for x in ins[t]]),
                outs[t][0].ctypes.data, outs[t][1].ctypes.data, C.byref(tk)))
            tickets.append(tk.value)
            if t >= 3:
                r = _abi.Report()
                pb.pipeline.check(lib.stitch_b200_wait(b.handle, tickets[t - 3], C.byref(r)))
                reps[t - 3] = r
        for t in range(4, 7):
            r = _abi.Report()
            pb.pipeline.check(lib.stitch_b200_wait(b.handle, tickets[t], C.byref(r)))
            reps[t] = r
        for t in range(7):
            np.testing.assert_array_equal(outs[t][0], want[t].panorama.data)
            np.testing.assert_array_equal(outs[t][1], want[t].panorama.mask)
            assert reps[t].frame_index == t
            assert list(reps[t].threshold_m1) == list(want[t].report.threshold_m1)
    finally:
        b.close()


@pytest.mark.parametrize("kind", ["ring", "chain"])
def test_masked_extension_rigs_parity(kind):
    """Masked inputs (Frame::mask) on the extension rigs the reference cannot
    run -- the 6-camera cylindrical 360-degree ring and a 4-view chain --
    against the extended oracle: masked first frames set the pair geometry,
    every frame's panorama / mask / report is identical, and a fully masked
    frame fails with EmptyProjection on both sides with the temporal state
    untouched (the frames after it still agree)."""
    from tests.golden.masks import input_mask

    if kind == "ring":
        spec = pb.SynthSpec(views=6, width=256, height=144, frames=5, rig="ring",
                            color_casts=[(1.0 - 0.04 * v, 1.0, 1.0 + 0.03 * v) for v in range(6)])
        sc = pb.SynthScene(spec)
        masked_views, empty = (0, 2, 3), (2, 3)
    else:
        sc = scene(views=4, width=200, height=150, frames=5,
                   casts=[(1.0, 1.0, 1.0), (0.9, 1.0, 1.1), (1.1, 0.95, 0.9), (0.95, 1.05, 1.0)])
        masked_views, empty = (1, 3), (3, 1)
    nv = sc.spec.views
    w, h = sc.spec.width, sc.spec.height

    def masks(t):
        out = []
        for v in range(nv):
            if v not in masked_views:
                out.append(None)
            elif (t, v) == empty:
                out.append(np.zeros((h, w), np.uint8))
            else:
                out.append(input_mask(31, v, t, w, h))
        return out

    def frames(t):
        ms = masks(t)
        return [pb.Frame(sc.render_view(v, t).data, ms[v]) for v in range(nv)]

    first = frames(0)
    state = pb.initialize(product_config(sc), first)
    ost = O.OracleState(oracle_config(sc), first_frames=[f.data for f in first],
                        first_masks=masks(0))
    try:
        assert state.canvas == ost.canvas
        for k, p in enumerate(state.pairs):
            view, partner, bounds = ost.pair(k)
            assert (p.view, p.partner, p.bounds) == (view, partner, bounds)
            np.testing.assert_array_equal(p.theta_i, ost.pair_weights(k))
        errors = 0
        for t in range(sc.spec.frames):
            fr = frames(t)
            if t == empty[0]:
                with pytest.raises(O.OracleError) as oe:
                    ost.process([f.data for f in fr], masks(t))
                with pytest.raises(pb.StitchError) as ge:
                    pb.process_frame(state, fr)
                assert O.ERROR_NAMES[oe.value.code] == "EmptyProjection"
                assert ge.value.code == pb.ErrorCode.EmptyProjection
                errors += 1
                continue
            res = pb.process_frame(state, fr)
            odata, omask, orep = ost.process([f.data for f in fr], masks(t))
            rep = res.report
            np.testing.assert_array_equal(res.panorama.mask, omask)
            assert maxdiff(res.panorama.data, odata) == 0, t
            for k in range(len(state.pairs)):
                np.testing.assert_array_equal(rep.color_matrices[k],
                                              np.array(orep.m[k][:]).reshape(3, 3))
                assert rep.rank_deficient[k] == bool(orep.rank_deficient[k])
            assert rep.threshold_m1 == list(orep.threshold_m1)
            assert rep.threshold_m2 == list(orep.threshold_m2)
            assert rep.frame_index == orep.frame_index
        assert errors == 1
    finally:
        state.close()
        ost.close()
        sc.close()
