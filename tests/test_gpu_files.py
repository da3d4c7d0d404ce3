"""File-to-file sequence runs (stitch_b200_run_files, the run_sequence of
pipeline.cpp:364-412 over numbered PPM sequences): the written panoramas
equal the oracle's frame for frame, the reports follow the frame order, and
bad inputs fail like the reference (IoError / InputMismatch)."""
import os

import numpy as np
import pytest

import oracle as O
import paper_2308_09209_b200 as pb
from paper_2308_09209_b200 import ErrorCode, StitchError
from tests.helpers import frames_at, oracle_config, product_config, scene

pytestmark = pytest.mark.gpu


def write_views(sc, root, frames, png_views=()):
    dirs = []
    for v in range(sc.spec.views):
        d = os.path.join(root, f"view{v}")
        os.makedirs(d, exist_ok=True)
        ext = ".png" if v in png_views else ".ppm"
        for t in range(frames):
            pb.write_image(os.path.join(d, pb.sequence_name("cam", t, ext)), sc.render_view(v, t))
        dirs.append(d)
    return dirs


def test_run_files_matches_oracle(tmp_path):
    sc = scene(views=3, width=200, height=150, frames=7,
               casts=[(0.9, 1, 1), (1, 1, 1), (1, 0.95, 1.1)],
               flicker=[pb.FlickerEvent(frame=3, view=2, gains=(1.2, 1.1, 0.9))])
    dirs = write_views(sc, str(tmp_path / "in"), 7)
    state = pb.initialize(product_config(sc), frames_at(sc, 0))
    ost = O.OracleState(oracle_config(sc))
    try:
        out = str(tmp_path / "out")
        res = pb.run_files(state, dirs, out, "pano")
        assert res.frames == 7 and len(res.reports) == 7
        assert sorted(os.listdir(out)) == [pb.sequence_name("pano", t, ".ppm") for t in range(7)]
        for t in range(7):
            odata, _, orep = ost.process([f.data for f in frames_at(sc, t)])
            got = pb.read_ppm(os.path.join(out, pb.sequence_name("pano", t, ".ppm")))
            np.testing.assert_array_equal(got.data, odata)
            assert res.reports[t].frame_index == t
            for k in range(len(state.pairs)):
                np.testing.assert_array_equal(res.reports[t].color_matrices[k],
                                              np.array(orep.m[k][:]).reshape(3, 3))
        assert res.fps() > 0
    finally:
        state.close()
        ost.close()


def test_run_files_png_in_and_out(tmp_path):
    """PNG sources (one view) and PNG panoramas with the mask as alpha."""
    sc = scene(views=2, width=160, height=120, frames=3, casts=[(1, 1, 1), (0.9, 1, 1.1)])
    dirs = write_views(sc, str(tmp_path / "in"), 3, png_views=(1,))
    state = pb.initialize(product_config(sc), frames_at(sc, 0))
    ost = O.OracleState(oracle_config(sc))
    try:
        out = str(tmp_path / "out")
        res = pb.run_files(state, dirs, out, "pano", ext=".png")
        assert res.frames == 3
        for t in range(3):
            odata, omask, _ = ost.process([f.data for f in frames_at(sc, t)])
            got = pb.read_png(os.path.join(out, pb.sequence_name("pano", t, ".png")))
            np.testing.assert_array_equal(got.mask if got.mask is not None else
                                          np.ones_like(omask), omask)
            np.testing.assert_array_equal(got.data, odata)
    finally:
        state.close()
        ost.close()


def test_run_files_limits_and_errors(tmp_path):
    sc = scene(views=2, width=160, height=120, frames=4)
    dirs = write_views(sc, str(tmp_path / "in"), 4)
    # a view with fewer frames bounds the run; max_frames bounds it further
    os.remove(os.path.join(dirs[1], pb.sequence_name("cam", 3, ".ppm")))
    state = pb.initialize(product_config(sc), frames_at(sc, 0))
    try:
        assert pb.run_files(state, dirs, None).frames == 3
        assert pb.run_files(state, dirs, None, max_frames=2).frames == 2
        # wrong frame size -> InputMismatch, and the context stays usable
        pb.write_ppm(os.path.join(dirs[0], pb.sequence_name("cam", 1, ".ppm")),
                     pb.Frame(np.zeros((10, 10, 3), np.uint8)))
        with pytest.raises(StitchError) as e:
            pb.run_files(state, dirs, None)
        assert e.value.code == ErrorCode.InputMismatch
        pb.process_frame(state, frames_at(sc, 0))
        # a transparent PNG source is a masked frame (image_io.cpp:120-127): it runs
        # with its mask (stitch_b200_submit_masked)
        f0 = frames_at(sc, 0)[0]
        mask = np.ones((120, 160), np.uint8)
        mask[5, 7] = 0
        mask[40:60, 70:90] = 0
        pb.write_png(os.path.join(dirs[0], pb.sequence_name("cam", 1, ".png")),
                     pb.Frame(f0.data, mask))
        os.remove(os.path.join(dirs[0], pb.sequence_name("cam", 1, ".ppm")))
        assert pb.run_files(state, dirs, None).frames == 3
        # a corrupt file -> IoError; a missing directory -> IoError
        open(os.path.join(dirs[0], pb.sequence_name("cam", 1, ".png")), "wb").close()
        with pytest.raises(StitchError) as e:
            pb.run_files(state, dirs, None)
        assert e.value.code == ErrorCode.IoError
        with pytest.raises(StitchError) as e:
            pb.run_files(state, [dirs[1], str(tmp_path / "missing")], None)
        assert e.value.code == ErrorCode.IoError
    finally:
        state.close()
