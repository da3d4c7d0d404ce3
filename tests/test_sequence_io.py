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


# ---- PNG (image_io.cpp:87-165), restated on zlib ----------------------------
import struct
import zlib


def _png_bytes(w, h, ctype, depth, rows, plte=None, trns=None, interlace=0):
    """A minimal PNG encoder (filter bytes given per row in `rows`)."""
    def chunk(t, d):
        return struct.pack(">I", len(d)) + t + d + struct.pack(">I", zlib.crc32(t + d) & 0xffffffff)
    out = b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, depth, ctype, 0, 0,
                                                            interlace))
    if plte is not None:
        out += chunk(b"PLTE", bytes(plte))
    if trns is not None:
        out += chunk(b"tRNS", bytes(trns))
    out += chunk(b"IDAT", zlib.compress(b"".join(rows)))
    return out + chunk(b"IEND", b"")


def test_png_round_trips_pixels_and_mask(tmp_path):
    # test_imaging.cpp:234-254: plain RGB round trip without a mask; a masked
    # frame writes RGBA and reads back the same mask and valid pixels
    rng = np.random.default_rng(4)
    f = rng.integers(0, 256, (19, 23, 3), dtype=np.uint8)
    pb.write_png(tmp_path / "plain.png", pb.Frame(f))
    g = pb.read_png(tmp_path / "plain.png")
    np.testing.assert_array_equal(g.data, f)
    assert g.mask is None
    m = (rng.random((19, 23)) >= 0.3).astype(np.uint8)
    pb.write_png(tmp_path / "masked.png", pb.Frame(f, m))
    h = pb.read_png(tmp_path / "masked.png")
    assert h.mask is not None
    np.testing.assert_array_equal(h.mask, m)
    np.testing.assert_array_equal(h.data[m == 1], f[m == 1])
    # the files are standard PNG: zlib-decodable, colour types 2 and 6
    raw = (tmp_path / "masked.png").read_bytes()
    assert raw[:8] == b"\x89PNG\r\n\x1a\n" and raw[12:16] == b"IHDR" and raw[25] == 6
    assert (tmp_path / "plain.png").read_bytes()[25] == 2


def test_png_decodes_filters_depths_and_colour_types(tmp_path):
    rng = np.random.default_rng(7)
    w, h = 9, 5
    rgb = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    # every filter type on 8-bit RGB (encoded by hand: Sub, Up, Average, Paeth)
    def filt(ft, row, prev, bpp):
        out = bytearray()
        for i, x in enumerate(row):
            a = row[i - bpp] if i >= bpp else 0
            b = prev[i]
            c = prev[i - bpp] if i >= bpp else 0
            p = a + b - c
            pa, pb_, pc = abs(p - a), abs(p - b), abs(p - c)
            pr = a if pa <= pb_ and pa <= pc else (b if pb_ <= pc else c)
            pred = [0, a, b, (a + b) // 2, pr][ft]
            out.append((x - pred) & 0xff)
        return bytes([ft]) + bytes(out)
    rows, prev = [], bytes(w * 3)
    for y in range(h):
        row = rgb[y].tobytes()
        rows.append(filt(y % 5, row, prev, 3))
        prev = row
    (tmp_path / "f.png").write_bytes(_png_bytes(w, h, 2, 8, rows))
    np.testing.assert_array_equal(pb.read_png(tmp_path / "f.png").data, rgb)
    # 16-bit RGB keeps the high byte (png_set_strip_16)
    rgb16 = rng.integers(0, 65536, (h, w, 3), dtype=np.uint16)
    rows = [b"\x00" + rgb16[y].astype(">u2").tobytes() for y in range(h)]
    (tmp_path / "d16.png").write_bytes(_png_bytes(w, h, 2, 16, rows))
    np.testing.assert_array_equal(pb.read_png(tmp_path / "d16.png").data, (rgb16 >> 8).astype(np.uint8))
    # 4-bit grey expands by 17 and replicates to RGB (png_set_expand + gray_to_rgb)
    grey = rng.integers(0, 16, (h, w), dtype=np.uint8)
    rows = []
    for y in range(h):
        px = list(grey[y]) + [0]
        rows.append(b"\x00" + bytes((px[2 * i] << 4) | px[2 * i + 1] for i in range((w + 1) // 2)))
    (tmp_path / "g4.png").write_bytes(_png_bytes(w, h, 0, 4, rows))
    got = pb.read_png(tmp_path / "g4.png").data
    np.testing.assert_array_equal(got, np.repeat((grey * 17)[..., None], 3, axis=2))
    # 8-bit palette with tRNS: entry 1 transparent -> masked
    pal = [10, 20, 30, 40, 50, 60, 70, 80, 90]
    idx = rng.integers(0, 3, (h, w), dtype=np.uint8)
    rows = [b"\x00" + idx[y].tobytes() for y in range(h)]
    (tmp_path / "p.png").write_bytes(_png_bytes(w, h, 3, 8, rows, plte=pal, trns=[255, 0]))
    fr = pb.read_png(tmp_path / "p.png")
    np.testing.assert_array_equal(fr.data, np.array(pal, np.uint8).reshape(3, 3)[idx])
    np.testing.assert_array_equal(fr.mask, (idx != 1).astype(np.uint8))
    # grey + alpha: alpha 0 -> invalid
    ga = np.stack([grey * 17, (grey % 2) * 255], axis=-1).astype(np.uint8)
    rows = [b"\x00" + ga[y].tobytes() for y in range(h)]
    (tmp_path / "ga.png").write_bytes(_png_bytes(w, h, 4, 8, rows))
    np.testing.assert_array_equal(pb.read_png(tmp_path / "ga.png").mask, (grey % 2).astype(np.uint8))


@pytest.mark.parametrize("mutate,what", [
    (lambda b: b[:8] + b[8:20] + bytes([b[20] ^ 1]) + b[21:], "CRC"),
    (lambda b: b"\x89PNX" + b[4:], "not a PNG"),
    (lambda b: b[:40], "truncated"),
])
def test_png_malformed_is_io_error(tmp_path, mutate, what):
    good = _png_bytes(2, 2, 2, 8, [b"\x00" + bytes(6)] * 2)
    p = tmp_path / "bad.png"
    p.write_bytes(mutate(good))
    with pytest.raises(StitchError) as e:
        pb.read_png(p)
    assert e.value.code == ErrorCode.IoError


def test_png_interlaced_is_rejected(tmp_path):
    p = tmp_path / "i.png"
    p.write_bytes(_png_bytes(2, 2, 2, 8, [b"\x00" + bytes(6)] * 2, interlace=1))
    with pytest.raises(StitchError) as e:
        pb.read_png(p)
    assert e.value.code == ErrorCode.IoError and "interlaced" in str(e.value)


def test_png_huge_header_is_rejected_before_allocating(tmp_path):
    """a crafted IHDR (2^20 x 2^20 pixels) fails with IoError instead of a
    multi-terabyte allocation that would throw through the C ABI"""
    p = tmp_path / "huge.png"
    p.write_bytes(_png_bytes(1 << 20, 1 << 20, 2, 8, [b"\x00" + bytes(6)]))
    with pytest.raises(StitchError) as e:
        pb.read_png(p)
    assert e.value.code == ErrorCode.IoError and "2^31" in str(e.value)


def test_sequence_listing_mixes_png_and_ppm(tmp_path):
    # test_imaging.cpp:257-269 with PNG files
    for i in [2, 0, 1]:
        pb.write_png(tmp_path / pb.sequence_name("frame", i), pb.Frame(np.full((4, 4, 3), 7, np.uint8)))
    names = [os.path.basename(f) for f in pb.list_sequence(tmp_path)]
    assert names == ["frame_000000.png", "frame_000001.png", "frame_000002.png"]
    assert pb.read_image(tmp_path / names[1]).data.shape == (4, 4, 3)
