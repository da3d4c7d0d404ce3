"""GPU quality metrics (metrics.cpp:9-155; the paper's Tables 2-3) against the
CPU oracle: psnr / ssim of arbitrary frames, the per-pair colour-transfer
quality of the stitching pipeline, and the 2D-M vs 3D-M comparison."""
import numpy as np
import pytest

import oracle as O
import paper_2308_09209_b200 as pb
from tests.helpers import frames_at, oracle_config, product_config, scene

pytestmark = pytest.mark.gpu


def _frames(seed, w, h, drop=0.0, corner=False):
    rng = np.random.default_rng(seed)
    a = rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
    b = ((a.astype(np.int32) * 3 + rng.integers(0, 256, size=(h, w, 3))) // 4).astype(np.uint8)
    ma = (rng.random((h, w)) >= drop).astype(np.uint8) if drop else None
    mb = None
    if corner:
        mb = np.ones((h, w), np.uint8)
        mb[: h // 3, : w // 3] = 0
    return a, ma, b, mb


@pytest.mark.parametrize("w,h,drop,corner", [(64, 48, 0.0, False), (200, 120, 0.05, True),
                                             (11, 11, 0.0, False), (517, 301, 0.0, True)])
def test_psnr_ssim_bit_exact_vs_oracle(w, h, drop, corner):
    a, ma, b, mb = _frames(w * h, w, h, drop, corner)
    fa, fb = pb.Frame(a, ma), pb.Frame(b, mb)
    assert pb.psnr(fa, fb) == O.psnr(a, ma, b, mb)
    # (a random per-pixel drop leaves no fully valid 11x11 window: SSIM on
    # the corner-masked pair only)
    assert pb.ssim(pb.Frame(a), fb) == O.ssim(a, None, b, mb)
    assert pb.psnr(fa, fa) == float("inf")
    assert pb.ssim(pb.Frame(a), pb.Frame(a)) == 1.0


def test_metric_errors():
    a = np.zeros((10, 20, 3), np.uint8)
    with pytest.raises(pb.StitchError):
        pb.ssim(pb.Frame(a), pb.Frame(a))  # TooSmall
    with pytest.raises(pb.StitchError):
        pb.psnr(pb.Frame(a, np.zeros((10, 20), np.uint8)), pb.Frame(a))  # EmptyRegion


def test_pair_quality_matches_oracle_crops():
    """Tables 2-3 columns computed on the device-resident overlap crops equal
    the oracle's metrics on its own warped crops and colour matrix."""
    sc = scene(views=2, width=160, height=120, frames=4, casts=[(1, 1, 1), (0.8, 1.0, 1.15)])
    cfg = product_config(sc)
    state = pb.initialize(cfg, frames_at(sc, 0))
    ost = O.OracleState(oracle_config(sc, keep_debug=1))
    for t in range(4):
        frames = frames_at(sc, t)
        pb.process_frame(state, frames)
        _, _, rep = ost.process([f.data for f in frames])
        view, partner, (x0, y0, x1, y1) = ost.pair(0)
        sv, smask = ost.last_warped(view)
        rv, rmask = ost.last_warped(partner)
        src, sm = sv[y0:y1, x0:x1], smask[y0:y1, x0:x1]
        ref, rm = rv[y0:y1, x0:x1], rmask[y0:y1, x0:x1]
        m = np.array(rep.m[0][:]).reshape(3, 3)
        cor = O.apply_color_matrix_rows(src, sm, m)
        want = (O.psnr(cor, sm, src, sm), O.psnr(cor, sm, ref, rm), O.ssim(cor, sm, ref, rm))
        got = state.pair_quality(0)
        assert got == want, (t, got, want)
    state.close()


def test_compare_methods_table_shape_and_flicker():
    """compare_methods_both: 2 methods x (frames + mu + sigma) rows; on a
    flicker-injected sequence the 3D-M window damps the frame-to-frame
    variation of the transfer quality (SPEC.md: sigma(window 3) <
    sigma(window 1), the directional analogue of Table 2)."""
    sc = scene(views=2, width=160, height=120, frames=6, casts=[(1, 1, 1), (0.85, 1.0, 1.1)],
               flicker=[pb.FlickerEvent(frame=3, view=1, gains=(1.3, 1.2, 1.25))])
    cfg = product_config(sc)
    views = [[sc.render_view(v, t) for t in range(6)] for v in range(2)]
    rows = pb.compare_methods(cfg, views, pair=0, scene_id="flicker")
    assert [r.method for r in rows] == ["2D-M"] * 8 + ["3D-M"] * 8
    assert [r.frame_label for r in rows[:8]] == ["1", "2", "3", "4", "5", "6", "mu", "sigma"]
    s2 = next(r for r in rows if r.method == "2D-M" and r.frame_label == "sigma")
    s3 = next(r for r in rows if r.method == "3D-M" and r.frame_label == "sigma")
    assert s3.psnr_vs_source < s2.psnr_vs_source
    # frame rows equal the pair quality of an independent run
    state = pb.initialize(cfg, [s[0] for s in views])
    for t in range(6):
        pb.process_frame(state, [s[t] for s in views])
        q = state.pair_quality(0)
        r = rows[8 + t]
        assert (r.psnr_vs_source, r.psnr_vs_reference, r.ssim_vs_reference) == q
    state.close()
