"""Deterministic input masks (Frame::mask, frame.hpp:44-47: 0/1 per pixel) for
the masked-input golden cases: what a PNG source with an alpha channel hands
the reference (image_io.cpp:120-127).  Plain numpy integer arithmetic, so the
same bytes on every machine; tests/test_ref_pin.py also checks their digests.

Per (seed, view, frame): a moving elliptical hole, a cut strip along one
border (view-dependent side), and ~1 % scattered single-pixel holes.  A spec
may leave some views or frames unmasked (None): mixed inputs."""
import numpy as np


def _hash(seed, view, frame, salt):
    x = (seed * 0x9E3779B1 + view * 0x85EBCA77 + frame * 0xC2B2AE3D + salt * 0x27D4EB2F) & 0xFFFFFFFF
    x ^= x >> 15
    x = (x * 0x2C1B3C6D) & 0xFFFFFFFF
    x ^= x >> 12
    return x


def input_mask(seed, view, frame, width, height):
    yy, xx = np.mgrid[0:height, 0:width]
    m = np.ones((height, width), np.uint8)
    # moving elliptical hole
    cx = (_hash(seed, view, 0, 1) % width + 7 * frame) % width
    cy = (_hash(seed, view, 0, 2) % height + 3 * frame) % height
    rx, ry = max(3, width // 10), max(3, height // 8)
    m[((xx - cx) * ry) ** 2 + ((yy - cy) * rx) ** 2 <= (rx * ry) ** 2] = 0
    # cut strip along one border
    side = view % 4
    cut = max(1, width // 40)
    if side == 0:
        m[:, :cut] = 0
    elif side == 1:
        m[:, width - cut:] = 0
    elif side == 2:
        m[:max(1, height // 40), :] = 0
    else:
        m[height - max(1, height // 40):, :] = 0
    # scattered single-pixel holes (~1 %)
    h = (xx.astype(np.uint64) * np.uint64(73856093) ^ yy.astype(np.uint64) * np.uint64(19349663)
         ^ np.uint64(_hash(seed, view, frame, 3)))
    m[(h % np.uint64(97)) == 0] = 0
    return m


def case_masks(spec, view, frame, width, height):
    """spec: {"seed": s, "views": [masked view ids], "skip_frames": [...],
    "empty": [[frame, view], ...]} -> mask or None; an "empty" entry is a
    fully masked frame (a PNG whose alpha is 0 everywhere)."""
    if spec is None or view not in spec["views"] or frame in spec.get("skip_frames", []):
        return None
    if [frame, view] in [list(e) for e in spec.get("empty", [])]:
        return np.zeros((height, width), np.uint8)
    return input_mask(spec["seed"], view, frame, width, height)
