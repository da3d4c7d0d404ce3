"""Host-side logic on CPU: the synthetic scene generator (input side of the
path, synth.cpp restated) and the N-view rig/pair extension."""
import numpy as np
import pytest

import paper_2308_09209_b200 as pb
from tests.helpers import scene


def test_yaw_rig_matches_reference_shape():
    # synth.cpp:71 reference_ = views == 3 ? 1 : 0; focal 0.9 * width
    sc2 = scene(views=2, width=640, height=480, obj=False)
    sc3 = scene(views=3, width=640, height=480, obj=False)
    assert sc2.reference_view() == 0 and sc3.reference_view() == 1
    c = sc2.config_c()
    assert c.cams[0].fx == pytest.approx(0.9 * 640)
    assert c.cams[0].cx == 320.0 and c.cams[0].cy == 240.0
    # the reference camera looks straight at the plane from z = -500
    assert list(c.cams[0].rotation) == [1, 0, 0, 0, 1, 0, 0, 0, 1]
    assert list(c.cams[0].translation) == [0.0, 0.0, 500.0]


def test_render_is_deterministic_and_textured():
    sc = scene(views=2, width=96, height=64)
    a = sc.render_view(1, 2).data
    b = sc.render_view(1, 2, threads=1).data
    np.testing.assert_array_equal(a, b)
    # value-noise texture in [20, 235] (synth.cpp:48-58)
    assert a.min() >= 20 and a.max() <= 235 and a.std() > 5


def test_color_casts_and_flicker_gains():
    base = scene(views=2, width=64, height=48, obj=False)
    cast = scene(views=2, width=64, height=48, obj=False, casts=[(1, 1, 1), (0.5, 1, 1)],
                 flicker=[pb.FlickerEvent(frame=1, view=1, gains=(1, 1, 0.5))])
    a = base.render_view(1, 1).data.astype(float)
    b = cast.render_view(1, 1).data.astype(float)
    assert np.abs(b[..., 0] - np.round(a[..., 0] * 0.5)).max() <= 1
    assert np.abs(b[..., 2] - np.round(a[..., 2] * 0.5)).max() <= 1
    np.testing.assert_array_equal(b[..., 1], a[..., 1])


def test_yaw_rig_rejects_more_than_three_views():
    with pytest.raises(pb.StitchError):
        pb.SynthScene(pb.SynthSpec(views=4, rig="yaw"))


def test_strip_rig_overlap_fraction():
    sc = scene(views=4, width=320, height=240, obj=False)
    assert sc.reference_view() == 1
    c = sc.config_c()
    # toe-in yaw grows by strip_yaw per step; cameras translate along x
    xs = [c.cams[v].translation[0] for v in range(4)]
    assert len(set(np.round(xs, 6))) == 4


def test_parallax_object_moves():
    sc = scene(views=2, width=128, height=96)
    a = sc.render_view(0, 0).data
    b = sc.render_view(0, 3).data
    assert (a != b).any()
    still = scene(views=2, width=128, height=96, obj=False)
    np.testing.assert_array_equal(still.render_view(0, 0).data, still.render_view(0, 3).data)
