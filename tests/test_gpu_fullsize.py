"""Parity at BASELINE.json's full sizes: the bench's own synthetic inputs
(4x1080p C2 across the flicker event, the 6-camera 360-degree ring C3, the
8x4K C4) through the C ABI against the CPU oracle on the box's host cores.

Contract tolerances (BASELINE.json north_star) are asserted, and the stricter
bit-exact expectation as well; tests/fullsize.py produces the same per-stage
max-abs-diff numbers that scripts/parity_report.py records in profiles/.
"""
import pytest

from tests.fullsize import run_config

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("key", ["c2", "c3", "c4"])
def test_full_size_config_parity(key):
    geom, frames, info = run_config(key)
    assert geom, f"{key}: init geometry differs from the oracle"
    assert len(frames) == info["frames"]
    for t, d in enumerate(frames):
        # contract tolerances
        assert d["color_matrix_max_rel"] <= 1e-4, (key, t, d)
        assert d["rank_flags_equal"], (key, t, d)
        assert d["flow_max_abs_px"] <= 1e-3, (key, t, d)
        assert d["panorama_max_abs_lsb"] <= 1, (key, t, d)
        assert d["mask_equal"] and d["thresholds_equal"] and d["frame_index_equal"], (key, t, d)
        # bit-exact expectation
        assert d["color_matrix_max_rel"] == 0.0 and d["flow_max_abs_px"] == 0.0, (key, t, d)
        assert d["panorama_max_abs_lsb"] == 0, (key, t, d)
