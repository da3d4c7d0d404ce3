"""GPU feature refinement (features.cpp, pipeline.cpp:114-179, 241-255)
against the CPU oracle: detection + description and matching kernels on
synthetic frames, then the whole refined initialize() and the frames it
stitches."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
import paper_2308_09209_b200 as pb
from paper_2308_09209_b200 import _abi
from tests.helpers import frames_at, oracle_config, product_config, scene

pytestmark = pytest.mark.gpu


def _lib():
    return _abi.load()


def gpu_detect(img, region, thr=2e-4, cap=20000):
    h, w = img.shape[:2]
    kp = np.zeros((cap, 4), np.float64)
    desc = np.zeros((cap, 64), np.float32)
    reg = (C.c_int * 4)(*region)
    n = _lib().stitch_b200_debug_detect(w, h, np.ascontiguousarray(img).ctypes.data, reg, thr, cap,
                                        kp.ctypes.data, desc.ctypes.data)
    assert n >= 0, n
    return [tuple(r) for r in kp[:n]], desc[:n]


def _texture(seed, w, h, block=4):
    rng = np.random.default_rng(seed)
    img = (rng.random((h // block + 1, w // block + 1, 3)) * 255).astype(np.uint8)
    img = np.repeat(np.repeat(img, block, axis=0), block, axis=1)[:h, :w]
    return np.ascontiguousarray(img)


@pytest.mark.parametrize("seed,region", [(1, (0, 0, 160, 120)), (2, (10, 7, 150, 101)),
                                         (3, (40, 30, 120, 90))])
def test_detect_describe_bit_exact(seed, region):
    img = _texture(seed, 160, 120)
    img[:, :20] = 0  # an invalid (zero) strip like a warped view's border
    kg, dg = gpu_detect(img, region)
    ko = O.detect(img, None, region)
    assert kg == ko
    np.testing.assert_array_equal(dg, O.describe(img, None, ko))


def test_match_bit_exact():
    a = _texture(5, 200, 150)
    b = np.roll(a, (3, 5), axis=(0, 1))
    ka, da = gpu_detect(a, (0, 0, 200, 150))
    kb, db = gpu_detect(b, (0, 0, 200, 150))
    na, nb = len(ka), len(kb)
    best_b = np.zeros(na, np.int32)
    best_d = np.zeros(na, np.float64)
    best_a = np.zeros(nb, np.int32)
    pb.pipeline.check(_lib().stitch_b200_debug_match(
        np.ascontiguousarray(da).ctypes.data, na, np.ascontiguousarray(db).ctypes.data, nb, 0.8,
        best_b.ctypes.data, best_d.ctypes.data, best_a.ctypes.data))
    got = [(i, int(best_b[i]), float(best_d[i])) for i in range(na)
           if best_b[i] >= 0 and best_a[best_b[i]] == i]
    want = [(m[0], m[1], m[2]) for m in O.match(da, db, ka, kb, 0.8)]
    assert got == want and len(got) > 10


@pytest.mark.parametrize("views", [2, 3])
def test_refined_initialize_matches_oracle(views):
    """initialize() with refinement on coarse homographies (3 % focal
    perturbation): refined maps, warnings, pair geometry and the stitched
    frames equal the oracle's."""
    sc = scene(views=views, width=320, height=240, frames=3, focal_scale=1.03,
               casts=[(1, 1, 1), (0.9, 1.0, 1.1), (1.05, 1.0, 0.95)][:views])
    cfg = product_config(sc, refine=True, seed=11)
    first = frames_at(sc, 0)
    state = pb.initialize(cfg, first)
    ost = O.OracleState(oracle_config(sc, refine=True, seed=11), [f.data for f in first])
    assert state.canvas == ost.canvas
    refined = 0
    for k, p in enumerate(state.pairs):
        assert p.refine_warning == ost.refine_warning(k)
        refined += not p.refine_warning
        view, partner, bounds = ost.pair(k)
        assert (p.view, p.partner, p.bounds) == (view, partner, bounds)
        np.testing.assert_array_equal(p.theta_i, ost.pair_weights(k))
    assert refined >= 1  # the perturbed maps were actually refined
    for v in range(views):
        _, inv = ost.maps(v)
        np.testing.assert_array_equal(state.inv_map(v), inv)
    unrefined = pb.initialize(product_config(sc), first)
    assert any(not np.array_equal(state.inv_map(v), unrefined.inv_map(v)) for v in range(views))
    for t in range(3):
        frames = frames_at(sc, t)
        res = pb.process_frame(state, frames)
        odata, omask, _ = ost.process([f.data for f in frames])
        np.testing.assert_array_equal(res.panorama.data, odata)
        np.testing.assert_array_equal(res.panorama.mask, omask)
    state.close()
    unrefined.close()


def test_refine_needs_frames():
    sc = scene(views=2, width=160, height=120, frames=1)
    cfg = product_config(sc, refine=True)
    c = pb.pipeline._config_to_c(cfg, [(160, 120)] * 2)
    h = C.c_void_p()
    rc = _lib().stitch_b200_initialize(C.byref(c), 0, C.byref(h))
    assert rc == pb.ErrorCode.ConfigurationError + 1


def test_run_sequence_rerefines():
    """refine.rerefine_every: the state is re-initialized from the current
    frames (pipeline.cpp:395-406) while the frame counter carries on; the
    re-refined geometry equals a fresh refined initialize() on those frames."""
    sc = scene(views=2, width=320, height=240, frames=4, focal_scale=1.03)
    cfg = product_config(sc, refine=True, seed=3)
    cfg.refine.rerefine_every = 2
    views = [[sc.render_view(v, t) for t in range(4)] for v in range(2)]
    res = pb.run_sequence(cfg, views)
    assert [r.frame_index for r in res.report.per_frame] == [0, 1, 2, 3]
    state = pb.initialize(cfg, [s[0] for s in views])
    for t in range(2):
        pb.process_frame(state, [s[t] for s in views])
    state.rerefine(cfg, [s[2] for s in views])
    fresh = pb.initialize(cfg, [s[2] for s in views])
    for v in range(2):
        np.testing.assert_array_equal(state.inv_map(v), fresh.inv_map(v))
    for a, b in zip(state.pairs, fresh.pairs):
        assert a.bounds == b.bounds and a.refine_warning == b.refine_warning
    r = pb.process_frame(state, [s[2] for s in views])
    assert r.report.frame_index == 2
    np.testing.assert_array_equal(r.panorama.data, res.panoramas[2].data)
    state.close()
    fresh.close()
