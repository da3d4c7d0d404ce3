"""Pins the CPU oracle to the reference's own known answers.

* proj/tests/test_imaging.cpp:34-191 (the one shipped unit test on this path:
  quantize, histogram, cdf, bilinear sampling), restated case by case;
* the SPEC.md operation examples for the per-frame path (the reference's
  unshipped tests), each cited by SPEC.md line.
Runs on CPU only.
"""
import numpy as np
import pytest

import oracle as O


def random_frame(rng, w, h, mask_drop=0.0):
    data = rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
    mask = None
    if mask_drop > 0:
        mask = (rng.random((h, w)) >= mask_drop).astype(np.uint8)
    return data, mask


def constant_frame(w, h, r, g, b):
    d = np.zeros((h, w, 3), np.uint8)
    d[..., 0], d[..., 1], d[..., 2] = r, g, b
    return d


# ---------------------------------------------------------------- test_imaging.cpp
def test_quantize_channel_rounds_half_away_and_clamps():  # test_imaging.cpp:34-41
    assert O.quantize_channel(0.5) == 1
    assert O.quantize_channel(1.5) == 2
    assert O.quantize_channel(2.4) == 2
    assert O.quantize_channel(254.5) == 255
    assert O.quantize_channel(-3.0) == 0
    assert O.quantize_channel(300.0) == 255


def test_histogram_constant_region():  # test_imaging.cpp:43-53
    f = constant_frame(16, 16, 128, 128, 128)
    bins, total = O.compute_histogram(f, None, (3, 3, 13, 13))
    assert total == 100
    for c in range(3):
        assert bins[c][128] == 100
        assert bins[c].sum() == 100


def test_histogram_two_pixels():  # test_imaging.cpp:55-64
    f = np.array([[[0, 0, 0], [255, 255, 255]]], np.uint8)
    bins, total = O.compute_histogram(f, None, (0, 0, 2, 1))
    assert total == 2
    for c in range(3):
        assert bins[c][0] == 1 and bins[c][255] == 1


def test_histogram_matches_tally_on_random_frames():  # test_imaging.cpp:66-86
    rng = np.random.default_rng(7)
    for trial in range(30):
        data, mask = random_frame(rng, 64, 64, 0.2 if trial % 3 == 0 else 0.0)
        x0, y0 = rng.integers(0, 41, size=2)
        r = (int(x0), int(y0), int(x0 + 1 + rng.integers(0, 41) % 23),
             int(y0 + 1 + rng.integers(0, 41) % 23))
        sub = data[r[1]:r[3], r[0]:r[2]]
        valid = np.ones(sub.shape[:2], bool) if mask is None else mask[r[1]:r[3], r[0]:r[2]] != 0
        expected = np.stack([np.bincount(sub[..., c][valid], minlength=256) for c in range(3)])
        if valid.sum() == 0:
            with pytest.raises(O.OracleError):
                O.compute_histogram(data, mask, r)
            continue
        bins, total = O.compute_histogram(data, mask, r)
        assert total == valid.sum()
        np.testing.assert_array_equal(bins, expected)


def test_histogram_rejects_empty_and_out_of_bounds():  # test_imaging.cpp:88-95
    f = constant_frame(8, 8, 1, 2, 3)
    with pytest.raises(O.OracleError):
        O.compute_histogram(f, None, (4, 4, 4, 6))
    with pytest.raises(O.OracleError):
        O.compute_histogram(f, None, (0, 0, 9, 8))
    with pytest.raises(O.OracleError):
        O.compute_histogram(np.zeros((8, 8, 3), np.uint8), np.zeros((8, 8), np.uint8),
                            (0, 0, 8, 8))


def test_cdf_closed_forms():  # test_imaging.cpp:97-138
    b = np.zeros((3, 256), np.int64)
    b[:, 0] = 10
    assert (O.cdf(b) == 1.0).all()
    u = np.full((3, 256), 4, np.int64)
    c = O.cdf(u)
    np.testing.assert_allclose(c[1], (np.arange(256) + 1) / 256.0, rtol=1e-12)
    assert c[0][255] == 1.0
    with pytest.raises(O.OracleError):
        O.cdf(np.zeros((3, 256), np.int64))


def test_bilinear_sampling_cases():  # test_imaging.cpp:140-174
    f = np.array([[[0, 0, 0], [100, 100, 100]]], np.uint8)
    ok, rgb = O.sample_bilinear(f, None, 1.0, 0.0)
    assert ok and rgb[0] == 100.0
    ok, rgb = O.sample_bilinear(f, None, 0.5, 0.0)
    assert ok and rgb[0] == pytest.approx(50.0)
    assert not O.sample_bilinear(f, None, -5.0, 0.0)[0]
    assert not O.sample_bilinear(f, None, 0.0, 3.0)[0]
    ok, rgb = O.sample_bilinear(f, None, -0.25, 0.0)
    assert ok and rgb[0] == pytest.approx(0.0)
    m = np.array([[[10, 10, 10], [200, 200, 200]]], np.uint8)
    mask = np.array([[1, 0]], np.uint8)
    ok, rgb = O.sample_bilinear(m, mask, 0.5, 0.0)
    assert ok and rgb[0] == pytest.approx(10.0)
    assert not O.sample_bilinear(m, np.array([[0, 0]], np.uint8), 0.5, 0.0)[0]


def test_bilinear_integer_coordinates_bit_exact():  # test_imaging.cpp:176-191
    rng = np.random.default_rng(23)
    for _ in range(10):
        data, _ = random_frame(rng, 17, 13)
        for y in range(13):
            for x in range(17):
                ok, rgb = O.sample_bilinear(data, None, float(x), float(y))
                assert ok
                assert (rgb == data[y, x].astype(np.float32)).all()


# ---------------------------------------------------------------- SPEC.md examples
def test_histogram_specification_examples():
    rng = np.random.default_rng(3)
    h = rng.integers(1, 50, size=(3, 256))
    lut = O.histogram_specification(h, h)
    np.testing.assert_array_equal(lut, np.tile(np.arange(256), (3, 1)))
    ref = np.zeros((3, 256), np.int64)
    ref[:, 128] = 1000
    assert (O.histogram_specification(h, ref) == 128).all()
    src = np.full((3, 256), 2, np.int64)
    ref = np.zeros((3, 256), np.int64)
    ref[:, :128] = 4
    lut = O.histogram_specification(src, ref)
    assert (np.abs(lut.astype(int) - np.arange(256) // 2) <= 1).all()
    assert (np.diff(lut.astype(int), axis=1) >= 0).all()  # monotone


def test_solve_color_matrix_examples():
    rng = np.random.default_rng(5)
    x = rng.integers(0, 128, size=(500, 3)).astype(np.float64)
    m, _ = O.solve_color_matrix([(x, x)])
    np.testing.assert_allclose(m, np.eye(3), atol=1e-12)
    a = np.diag([0.5, 1.0, 2.0])
    m, _ = O.solve_color_matrix([(x, x @ a)])
    np.testing.assert_allclose(m, a, atol=1e-9)
    # stacked window of 3 entries recovering a full 3x3 A within 1e-6
    A = np.array([[0.9, 0.05, 0.0], [0.1, 1.1, -0.05], [0.0, 0.02, 0.8]])
    win = []
    for _ in range(3):
        xs = rng.integers(0, 200, size=(300, 3)).astype(np.float64)
        win.append((xs, xs @ A))
    m, _ = O.solve_color_matrix(win)
    np.testing.assert_allclose(m, A, rtol=1e-6, atol=1e-9)
    same = np.tile([[10.0, 20.0, 30.0]], (50, 1))
    with pytest.raises(O.OracleError) as e:
        O.solve_color_matrix([(same, same)])
    assert O.ERROR_NAMES[e.value.code] == "RankDeficient"


def test_apply_color_matrix_clamp():
    f = np.array([[[200, 10, 10]]], np.uint8)
    out = O.apply_color_matrix_rows(f, None, np.diag([2.0, 2.0, 2.0]))
    assert list(out[0, 0]) == [255, 20, 20]


def test_find_thresholds_examples():
    u = np.ones((3, 256), np.int64)
    m1, m2 = O.find_thresholds(u, 0.05)
    assert m1 == [12, 12, 12] and m2 == [243, 243, 243]
    b = np.zeros((3, 256), np.int64)
    b[:, 200] = 77
    m1, m2 = O.find_thresholds(b, 0.05)
    assert m1 == [200] * 3 and m2 == [200] * 3


def test_smooth_thresholds_examples():
    hist = [([10, 0, 0], [200, 200, 200]), ([13, 0, 0], [200, 200, 200]),
            ([16, 0, 0], [200, 200, 200])]
    m1, _ = O.smooth_thresholds(hist)
    assert m1[0] == 13
    m1, m2 = O.smooth_thresholds(hist[:1])
    assert m1 == [10, 0, 0] and m2 == [200, 200, 200]
    m1, _ = O.smooth_thresholds([([10, 0, 0], [9, 9, 9]), ([13, 0, 0], [9, 9, 9])])
    assert m1[0] == 9  # mean 11.5 -> 12 crosses m2 = 9 -> swapped
    # only the newest 3 entries count
    m1, _ = O.smooth_thresholds([([100, 0, 0], [200] * 3)] + hist)
    assert m1[0] == 13


def test_build_curve_examples():
    ident = np.tile(np.arange(256), (3, 1))
    np.testing.assert_array_equal(O.build_curve([0] * 3, [255] * 3, 1.0, 1.0), ident)
    np.testing.assert_array_equal(O.build_curve([40] * 3, [215] * 3, 1.0, 1.0), ident)
    lut = O.build_curve([40] * 3, [215] * 3, 2.2, 2.2).astype(int)
    assert (np.diff(lut, axis=1) >= 0).all()
    assert np.abs(np.diff(lut, axis=1)).max() <= 6
    assert lut[0][0] == 0 and lut[0][255] == 255
    # degenerate thresholds -> global line
    np.testing.assert_array_equal(O.build_curve([100] * 3, [100] * 3, 2.2, 2.2), ident)


def test_warp_examples():
    rng = np.random.default_rng(11)
    data, _ = random_frame(rng, 40, 30)
    out, mask = O.warp_frame(data, np.eye(3), 40, 30, 0.0, 0.0)
    np.testing.assert_array_equal(out, data)
    assert mask.all()
    # translation by (5, 0): content shifted 5 px, 5-px invalid strip
    h = np.array([[1.0, 0, 5.0], [0, 1.0, 0], [0, 0, 1.0]])
    out, mask = O.warp_frame(data, np.linalg.inv(h), 40, 30, 0.0, 0.0)
    np.testing.assert_array_equal(out[:, 5:], data[:, :35])
    assert (mask[:, :4] == 0).all() and mask[:, 5:].all()
    # 2x scale matches an independent 2x bilinear upsample within 1 level
    s = np.diag([2.0, 2.0, 1.0])
    out, mask = O.warp_frame(data, np.linalg.inv(s), 78, 58, 0.0, 0.0)
    ys, xs = np.mgrid[0:58, 0:78] / 2.0
    x0, y0 = np.floor(xs).astype(int), np.floor(ys).astype(int)
    ax, ay = xs - x0, ys - y0
    x1, y1 = np.minimum(x0 + 1, 39), np.minimum(y0 + 1, 29)
    d = data.astype(np.float64)
    ref = ((1 - ay)[..., None] * ((1 - ax)[..., None] * d[y0, x0] + ax[..., None] * d[y0, x1]) +
           ay[..., None] * ((1 - ax)[..., None] * d[y1, x0] + ax[..., None] * d[y1, x1]))
    assert np.abs(out.astype(int) - np.round(ref)).max() <= 1


def _texture(rng, w, h, scale=6):
    small = rng.random((h // scale + 3, w // scale + 3, 3))
    ys, xs = np.mgrid[0:h, 0:w] / scale
    x0, y0 = np.floor(xs).astype(int), np.floor(ys).astype(int)
    ax, ay = (xs - x0)[..., None], (ys - y0)[..., None]
    v = ((1 - ay) * ((1 - ax) * small[y0, x0] + ax * small[y0, x0 + 1]) +
         ay * ((1 - ax) * small[y0 + 1, x0] + ax * small[y0 + 1, x0 + 1]))
    return (30 + 190 * v).round().astype(np.uint8)


def test_flow_examples():
    rng = np.random.default_rng(2)
    a = _texture(rng, 96, 64)
    u, v = O.dense_flow(a, None, a, None)
    assert np.abs(u).max() < 0.1 and np.abs(v).max() < 0.1
    big = _texture(rng, 102, 64)
    a, b = big[:, 3:99], big[:, 0:96]  # b(x) = a(x - 3)
    u, v = O.dense_flow(a, None, b, None)
    inner = (slice(8, -8), slice(8, -8))
    assert 2.5 <= np.median(u[inner]) <= 3.5
    assert -0.5 <= np.median(v[inner]) <= 0.5
    flat = np.full((40, 40, 3), 128, np.uint8)
    u, v = O.dense_flow(flat, None, flat, None)
    assert np.abs(u).max() == 0 and np.abs(v).max() == 0
    with pytest.raises(O.OracleError):
        O.dense_flow(flat[:15], None, flat[:15], None)  # TooSmall


def test_blend_weights_examples():
    h, w = 20, 60
    mi = np.zeros((h, w), np.uint8)
    mj = np.zeros((h, w), np.uint8)
    mi[:, :40] = 1
    mj[:, 20:] = 1
    ti, tj = O.blend_weights(mi, mj, (20, 0, 40, 20))
    np.testing.assert_array_equal(ti + tj, np.ones_like(ti))
    assert ti[:, 0].min() == 1.0 and ti[:, -1].max() == 0.0  # own side -> 1
    assert np.abs(ti[:, 9:11] - 0.5).max() <= 0.06  # midline ~0.5


def test_fuse_and_compose_examples():
    rng = np.random.default_rng(9)
    ri, _ = random_frame(rng, 30, 20)
    rj, _ = random_frame(rng, 30, 20)
    mask = np.ones((20, 30), np.uint8)
    z = np.zeros((20, 30), np.float32)
    th = rng.random((20, 30)).astype(np.float32)
    out, m = O.flow_fuse((ri, mask), (rj, mask), z, z, z, z, th)
    ref = th[..., None] * ri.astype(np.float32) + (1 - th)[..., None] * rj.astype(np.float32)
    assert np.abs(out.astype(int) - np.round(ref)).max() <= 1 and m.all()
    out, _ = O.flow_fuse((ri, mask), (ri, mask), z, z, z, z, th)
    np.testing.assert_array_equal(out, ri)
    # compose: disjoint masks -> side-by-side copy
    a, _ = random_frame(rng, 30, 20)
    b, _ = random_frame(rng, 30, 20)
    ma = np.zeros((20, 30), np.uint8)
    mb = np.zeros((20, 30), np.uint8)
    ma[:, :15] = 1
    mb[:, 15:] = 1
    fused = (np.zeros((1, 1, 3), np.uint8), np.zeros((1, 1), np.uint8))
    out, m = O.compose_panorama((a, ma), (b, mb), fused, (0, 0, 1, 1))
    np.testing.assert_array_equal(out[:, :15], a[:, :15])
    np.testing.assert_array_equal(out[:, 15:], b[:, 15:])
    assert m.all()


# ---- quality metrics (metrics.cpp:9-155) ----
def _np_ssim(a, am, b, bm):
    """Independent windowed-loop SSIM restatement (numpy, different summation order)."""
    h, w = a.shape[:2]
    valid = np.ones((h, w), bool)
    if am is not None:
        valid &= am.astype(bool)
    if bm is not None:
        valid &= bm.astype(bool)
    lum = lambda d: np.where(valid, 0.299 * d[..., 0] + 0.587 * d[..., 1] + 0.114 * d[..., 2], 0.0)
    la, lb = lum(a.astype(np.float64)), lum(b.astype(np.float64))
    d = np.arange(11) - 5.0
    k = np.exp(-d * d / (2 * 1.5 * 1.5))
    k /= k.sum()
    g2 = np.outer(k, k)
    c1, c2 = (0.01 * 255) ** 2, (0.03 * 255) ** 2
    vals = []
    for y in range(5, h - 5):
        for x in range(5, w - 5):
            if not valid[y - 5:y + 6, x - 5:x + 6].all():
                continue
            pa, pb = la[y - 5:y + 6, x - 5:x + 6], lb[y - 5:y + 6, x - 5:x + 6]
            ma, mb = (g2 * pa).sum(), (g2 * pb).sum()
            va, vb = (g2 * pa * pa).sum() - ma * ma, (g2 * pb * pb).sum() - mb * mb
            cov = (g2 * pa * pb).sum() - ma * mb
            vals.append((2 * ma * mb + c1) * (2 * cov + c2) / ((ma * ma + mb * mb + c1) * (va + vb + c2)))
    return float(np.mean(vals))


def test_psnr_examples():
    rng = np.random.default_rng(21)
    a, _ = random_frame(rng, 40, 30)
    assert O.psnr(a, None, a, None) == float("inf")
    b = a.copy().astype(np.int16)
    b = np.where(b == 255, 254, b + 1).astype(np.uint8)  # every sample differs by exactly 1
    assert abs(O.psnr(a, None, b, None) - 20 * np.log10(255.0)) <= 1e-4
    c, cm = random_frame(rng, 40, 30, mask_drop=0.2)
    am = (rng.random((30, 40)) >= 0.1).astype(np.uint8)
    valid = cm.astype(bool) & am.astype(bool)
    d = a.astype(np.float64) - c.astype(np.float64)
    mse = (d[valid] ** 2).sum() / (3 * valid.sum())
    assert abs(O.psnr(a, am, c, cm) - 10 * np.log10(255.0 ** 2 / mse)) <= 1e-9
    assert O.psnr(a, am, c, cm) == O.psnr(c, cm, a, am)  # symmetric
    with pytest.raises(O.OracleError):
        O.psnr(a, None, a[:20], None)  # ShapeMismatch
    with pytest.raises(O.OracleError):
        O.psnr(a, np.zeros((30, 40), np.uint8), a, None)  # EmptyRegion


def test_ssim_examples():
    rng = np.random.default_rng(22)
    a, _ = random_frame(rng, 36, 28)
    assert abs(O.ssim(a, None, a, None) - 1.0) <= 1e-9
    zero = np.zeros((28, 36, 3), np.uint8)
    full = np.full((28, 36, 3), 255, np.uint8)
    c1 = (0.01 * 255) ** 2
    assert abs(O.ssim(zero, None, full, None) - c1 / (255.0 ** 2 + c1)) <= 1e-12
    b, _ = random_frame(rng, 36, 28)
    bm = np.ones((28, 36), np.uint8)
    bm[:9, :12] = 0  # an invalid corner: windows touching it are skipped
    b = ((a.astype(np.int32) * 3 + b) // 4).astype(np.uint8)  # correlated with a
    assert abs(O.ssim(a, None, b, bm) - _np_ssim(a, None, b, bm)) <= 1e-6
    with pytest.raises(O.OracleError):
        O.ssim(a[:10], None, a[:10], None)  # TooSmall


# ---- feature refinement (features.cpp) ----
def _disc(h=96, w=96, cx=40, cy=48, r=8):
    yy, xx = np.mgrid[:h, :w]
    img = np.full((h, w, 3), 255, np.uint8)
    img[(yy - cy) ** 2 + (xx - cx) ** 2 <= r * r] = 0
    return img


def test_detect_examples():
    flat = np.full((64, 64, 3), 128, np.uint8)
    assert O.detect(flat, None, (0, 0, 64, 64)) == []
    img = _disc()
    kps = O.detect(img, None, (0, 0, 96, 96))
    assert kps and abs(kps[0][0] - 40) <= 2 and abs(kps[0][1] - 48) <= 2
    assert 8 / 2.5 <= kps[0][2] <= 8 * 2  # detection sigma of the strongest blob vs radius 8
    assert kps == O.detect(img, None, (0, 0, 96, 96))  # deterministic
    resp = [k[3] for k in kps]
    assert resp == sorted(resp, reverse=True)
    with pytest.raises(O.OracleError):
        O.detect(img, None, (0, 0, 31, 96))  # RegionTooSmall


def test_describe_and_match_examples():
    rng = np.random.default_rng(31)
    img = (rng.random((120, 160, 3)) * 255).astype(np.uint8)
    img = np.repeat(np.repeat(img[::4, ::4], 4, axis=0), 4, axis=1)  # blocky texture
    kps = O.detect(img, None, (0, 0, 160, 120))
    d = O.describe(img, None, kps)
    assert np.allclose(np.linalg.norm(d, axis=1), 1.0, atol=1e-5)
    np.testing.assert_array_equal(d, O.describe(img.copy(), None, kps))
    m = O.match(d, d, kps, kps)
    assert len(m) == len(kps) and all(a == b for a, b, *_ in m)  # identity matching
    dup = np.concatenate([d, d[:1]])  # a duplicated descriptor fails the ratio test
    m2 = O.match(d[:1], dup, kps[:1], kps + kps[:1])
    assert m2 == []


def test_ransac_examples():
    rng = np.random.default_rng(32)
    pts = rng.random((60, 2)) * 600
    exact = [(x, y, 1.1 * x + 4, 1.0 * y - 2) for x, y in pts]
    sx, sy, tx, ty = O.ransac(exact, seed=7)
    assert abs(sx - 1.1) <= 1e-9 and abs(sy - 1.0) <= 1e-9
    assert abs(tx - 4) <= 1e-6 and abs(ty + 2) <= 1e-6
    noisy = list(exact)
    for i in range(0, 60, 5):  # 40 % uniform outliers
        noisy[i] = (pts[i][0], pts[i][1], rng.random() * 600, rng.random() * 600)
    for i in range(1, 60, 5):
        noisy[i] = (pts[i][0], pts[i][1], rng.random() * 600, rng.random() * 600)
    sx, sy, tx, ty = O.ransac(noisy, seed=7)
    assert abs(sx - 1.1) <= 0.01 and abs(sy - 1.0) <= 0.01
    assert abs(tx - 4) <= 0.5 and abs(ty + 2) <= 0.5
    perm = [noisy[i] for i in rng.permutation(60)]
    assert O.ransac(perm, seed=7) == O.ransac(noisy, seed=7)  # canonical order
    with pytest.raises(O.OracleError):
        O.ransac(exact[:1])  # InsufficientMatches
