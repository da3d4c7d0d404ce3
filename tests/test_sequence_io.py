"""Frame ingress / egress: the PPM I/O and sequence
helpers of proj/src/image_io.cpp:19-199 through the C ABI.  Host-only calls
(no GPU): round trips are bit-exact, header comments are skipped like
read_ppm_token, malformed files raise IoError like the reference."""
import os

import numpy as np
import pytest

import paper_2308_09209_b200 as pb
from paper_2308_09209_b200 import ErrorCode, StitchError


def test_ppm_round_trip_bit_exact(tmp_path):
    rng = np.random.default_rng(3)
    for w, h in [(1, 1), (7, 5), (640, 480)]:
        data = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
        p = tmp_path / f"f{w}.ppm"
        pb.write_ppm(p, pb.Frame(data))
        raw = p.read_bytes()
        assert raw.startswith(f"P6\n{w} {h}\n255\n".encode())  # image_io.cpp:81
        back = pb.read_ppm(p)
        assert back.data.shape == (h, w, 3)
        np.testing.assert_array_equal(back.data, data)


def test_ppm_header_comments_and_whitespace(tmp_path):
    data = np.arange(2 * 3 * 3, dtype=np.uint8).reshape(2, 3, 3)
    p = tmp_path / "c.ppm"
    p.write_bytes(b"P6\n# a comment\n3 # width\n  2\n#x\n255\n" + data.tobytes())
    np.testing.assert_array_equal(pb.read_ppm(p).data, data)


@pytest.mark.parametrize("content,what", [
    (b"P3\n1 1\n255\n000", "not a P6"),
    (b"P6\n1 1\n65535\n" + bytes(6), "header"),
    (b"P6\n0 1\n255\n", "header"),
    (b"P6\n2 2\n255\n" + bytes(5), "truncated"),
])
def test_ppm_malformed_is_io_error(tmp_path, content, what):
    p = tmp_path / "bad.ppm"
    p.write_bytes(content)
    with pytest.raises(StitchError) as e:
        pb.read_ppm(p)
    assert e.value.code == ErrorCode.IoError
    assert what in str(e.value)


def test_missing_file_and_unwritable_path(tmp_path):
    with pytest.raises(StitchError) as e:
        pb.read_ppm(tmp_path / "nope.ppm")
    assert e.value.code == ErrorCode.IoError
    with pytest.raises(StitchError) as e:
        pb.write_ppm(tmp_path / "no_dir" / "x.ppm", pb.Frame(np.zeros((1, 1, 3), np.uint8)))
    assert e.value.code == ErrorCode.IoError


def test_sequence_name_and_listing(tmp_path):
    assert pb.sequence_name("pano", 3) == "pano_000003.png"  # image_io.hpp:29
    assert pb.sequence_name("v", 123456, ".ppm") == "v_123456.ppm"
    for i in [2, 0, 10, 1]:
        pb.write_ppm(tmp_path / pb.sequence_name("cam", i, ".ppm"),
                     pb.Frame(np.full((1, 1, 3), i, np.uint8)))
    (tmp_path / "notes.txt").write_text("x")
    os.mkdir(tmp_path / "sub.ppm")  # directories are skipped
    names = [os.path.basename(f) for f in pb.list_sequence(tmp_path)]
    assert names == ["cam_000000.ppm", "cam_000001.ppm", "cam_000002.ppm", "cam_000010.ppm"]
    with pytest.raises(StitchError) as e:
        pb.list_sequence(tmp_path / "cam_000000.ppm")
    assert e.value.code == ErrorCode.IoError
