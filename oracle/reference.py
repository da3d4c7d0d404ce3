"""THE REFERENCE ITSELF, compiled -- test infrastructure only.

ctypes binding of oracle/_ref/libstitch_ref.so: the unmodified reference
sources (/root/reference/proj/src/*.cpp) compiled against the Eigen-subset
shim by oracle/ref/Makefile, behind the thin C ABI in oracle/ref/ref_harness.cpp.
tests/test_ref_pin.py uses it to pin oracle/stitch_oracle.c (the restatement
the GPU parity tests compare against) to the reference's own outputs, and
bench.py's `--impl reference` arm times it.  The product never imports it.

The library is built here (where /root/reference exists) and ships to the GPU
box as a prebuilt file; `available()` is False when neither holds.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libstitch_ref.so")
REF_SRC = "/root/reference/proj/src"
MAX = 16
OK = -1


class RefSpec(C.Structure):
    class _Flicker(C.Structure):
        _fields_ = [("frame", C.c_int), ("view", C.c_int), ("gains", C.c_double * 3)]

    _fields_ = [("seed", C.c_uint64), ("views", C.c_int), ("frames", C.c_int),
                ("width", C.c_int), ("height", C.c_int), ("overlap_fraction", C.c_double),
                ("n_casts", C.c_int), ("casts", (C.c_double * 3) * MAX),
                ("n_flicker", C.c_int), ("flicker", _Flicker * MAX),
                ("object_enabled", C.c_int), ("depth_fraction", C.c_double),
                ("half_size", C.c_double), ("position", C.c_double * 2),
                ("velocity", C.c_double * 2), ("perturb_focal_scale", C.c_double),
                ("perturb_principal_px", C.c_double)]


class RefOpts(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("gamma_dark", C.c_double),
                ("gamma_bright", C.c_double), ("target_black", C.c_int),
                ("target_white", C.c_int), ("levels", C.c_int), ("iterations", C.c_int),
                ("smoothness", C.c_double), ("window_capacity", C.c_int),
                ("fuse_weighting", C.c_int), ("threads", C.c_int), ("refine_enabled", C.c_int),
                ("refine_margin", C.c_double), ("ransac_iters", C.c_int),
                ("inlier_px", C.c_double), ("detect_threshold", C.c_double),
                ("match_ratio", C.c_double), ("rerefine_every", C.c_int)]


class RefReport(C.Structure):
    _fields_ = [("frame_index", C.c_long), ("n_pairs", C.c_int),
                ("m", (C.c_double * 9) * MAX), ("rank_deficient", C.c_int * MAX),
                ("m1", C.c_int * 3), ("m2", C.c_int * 3)]


_lib = None


def build() -> bool:
    """Compile the library when the reference sources are present (here)."""
    if not os.path.isdir(REF_SRC):
        return os.path.exists(LIB_PATH)
    subprocess.run(["make", "-s", "-j8", "-C", os.path.join(_HERE, "ref")], check=True)
    return True


def available() -> bool:
    return os.path.exists(LIB_PATH) or os.path.isdir(REF_SRC)


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if os.path.isdir(REF_SRC):
        build()
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    sigs = {
        "ref_last_error": (C.c_char_p, []),
        "ref_default_opts": (None, [P(RefOpts)]),
        "ref_scene_new": (C.c_void_p, [P(RefSpec), P(C.c_int)]),
        "ref_scene_free": (None, [C.c_void_p]),
        "ref_scene_reference": (C.c_int, [C.c_void_p]),
        "ref_scene_render": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
        "ref_scene_cameras": (C.c_int, [C.c_void_p, P(C.c_double)]),
        "ref_state_new": (C.c_void_p, [C.c_void_p, P(RefOpts), P(C.c_void_p), P(C.c_void_p),
                                        P(C.c_int)]),
        "ref_state_free": (None, [C.c_void_p]),
        "ref_state_canvas": (None, [C.c_void_p, P(C.c_int), P(C.c_int), P(C.c_double),
                                    P(C.c_double)]),
        "ref_state_map": (None, [C.c_void_p, C.c_int, P(C.c_double), P(C.c_double)]),
        "ref_state_n_pairs": (C.c_int, [C.c_void_p]),
        "ref_state_pair": (None, [C.c_void_p, C.c_int, P(C.c_int), P(C.c_int), P(C.c_int)]),
        "ref_state_pair_weights": (None, [C.c_void_p, C.c_int, P(C.c_float), P(C.c_float)]),
        "ref_process_sized": (C.c_int, [C.c_void_p, C.c_int, P(C.c_int), P(C.c_int),
                                        P(C.c_void_p), P(C.c_void_p), C.c_void_p, C.c_void_p,
                                        P(RefReport)]),
        "ref_dense_flow": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_int,
                                     P(C.c_float), P(C.c_float)]),
        "ref_warp_frame": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_void_p, P(C.c_double),
                                     C.c_int, C.c_int, C.c_double, C.c_double, C.c_void_p,
                                     C.c_void_p]),
        "ref_build_curve": (None, [P(C.c_int), P(C.c_int), C.c_double, C.c_double, C.c_int,
                                   C.c_int, C.c_void_p]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


class RefError(RuntimeError):
    def __init__(self, code: int):
        self.code = code
        super().__init__(f"reference error {code}: {lib().ref_last_error().decode()}")


def default_opts(**kw) -> RefOpts:
    """StitchConfig defaults (pipeline.hpp:17-45), then keyword overrides."""
    o = RefOpts()
    lib().ref_default_opts(C.byref(o))
    for k, v in kw.items():
        setattr(o, "lambda_" if k == "lam" else k, v)
    return o


def _mask_ptrs(masks, n):
    """NULL for no masks, else a per-view pointer table (NULL = unmasked view)."""
    if masks is None or all(m is None for m in masks):
        return None, []
    keep = [None if m is None else np.ascontiguousarray(m, np.uint8) for m in masks]
    return (C.c_void_p * n)(*[None if m is None else m.ctypes.data for m in keep]), keep


class Scene:
    """stitch::SynthScene (synth.hpp:47-86) -- the reference's own renderer."""

    def __init__(self, seed=1, views=2, frames=5, width=320, height=240, overlap=0.3,
                 casts=None, flicker=None, obj=None, focal_scale=1.0, principal_px=0.0):
        s = RefSpec()
        s.seed, s.views, s.frames, s.width, s.height = seed, views, frames, width, height
        s.overlap_fraction = overlap
        casts = casts or []
        s.n_casts = len(casts)
        for v, g in enumerate(casts):
            for c in range(3):
                s.casts[v][c] = float(g[c])
        flicker = flicker or []
        s.n_flicker = len(flicker)
        for i, f in enumerate(flicker):
            s.flicker[i].frame, s.flicker[i].view = f["frame"], f["view"]
            for c in range(3):
                s.flicker[i].gains[c] = float(f["gains"][c])
        o = obj or {}
        s.object_enabled = 1 if o.get("enabled", False) else 0
        s.depth_fraction = o.get("depth_fraction", 0.15)
        s.half_size = o.get("half_size", 40.0)
        s.position[0], s.position[1] = o.get("position", (0.0, 0.0))
        s.velocity[0], s.velocity[1] = o.get("velocity", (0.0, 0.0))
        s.perturb_focal_scale = focal_scale
        s.perturb_principal_px = principal_px
        self.spec = s
        err = C.c_int(OK)
        self._h = lib().ref_scene_new(C.byref(s), C.byref(err))
        if not self._h:
            raise RefError(err.value)
        self.views, self.width, self.height = views, width, height

    @property
    def reference(self) -> int:
        return lib().ref_scene_reference(self._h)

    def render(self, view: int, frame: int) -> np.ndarray:
        out = np.zeros((self.height, self.width, 3), np.uint8)
        rc = lib().ref_scene_render(self._h, view, frame, out.ctypes.data)
        if rc != OK:
            raise RefError(rc)
        return out

    def cameras(self):
        buf = (C.c_double * (16 * MAX))()
        n = lib().ref_scene_cameras(self._h, buf)
        return [tuple(buf[16 * v:16 * v + 16]) for v in range(n)]

    def close(self):
        if self._h:
            lib().ref_scene_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class State:
    """stitch::PipelineState from stitch::initialize (pipeline.cpp:209-257)."""

    def __init__(self, scene: Scene, opts: RefOpts, first_frames, first_masks=None):
        self._keep = [np.ascontiguousarray(f, np.uint8) for f in first_frames]
        ptrs = (C.c_void_p * len(self._keep))(*[f.ctypes.data for f in self._keep])
        mptrs, self._keep_m = _mask_ptrs(first_masks, len(self._keep))
        err = C.c_int(OK)
        self._h = lib().ref_state_new(scene._h, C.byref(opts), ptrs, mptrs, C.byref(err))
        if not self._h:
            raise RefError(err.value)
        w, h, ox, oy = C.c_int(), C.c_int(), C.c_double(), C.c_double()
        lib().ref_state_canvas(self._h, C.byref(w), C.byref(h), C.byref(ox), C.byref(oy))
        self.canvas = (w.value, h.value, ox.value, oy.value)

    def n_pairs(self) -> int:
        return lib().ref_state_n_pairs(self._h)

    def pair(self, k):
        v, rw = C.c_int(), C.c_int()
        b = (C.c_int * 4)()
        lib().ref_state_pair(self._h, k, C.byref(v), b, C.byref(rw))
        return v.value, tuple(b[:]), bool(rw.value)

    def pair_weights(self, k):
        _, b, _ = self.pair(k)
        ti = np.zeros((b[3] - b[1], b[2] - b[0]), np.float32)
        tj = np.zeros_like(ti)
        lib().ref_state_pair_weights(self._h, k, ti.ctypes.data_as(C.POINTER(C.c_float)),
                                     tj.ctypes.data_as(C.POINTER(C.c_float)))
        return ti, tj

    def maps(self, v):
        h, inv = (C.c_double * 9)(), (C.c_double * 9)()
        lib().ref_state_map(self._h, v, h, inv)
        return np.array(h[:]).reshape(3, 3), np.array(inv[:]).reshape(3, 3)

    def process(self, frames, masks=None):
        """frames: RGB8 arrays; masks: None or per frame None / (H, W) 0/1."""
        fs = [np.ascontiguousarray(f, np.uint8) for f in frames]
        n = len(fs)
        ws = (C.c_int * n)(*[f.shape[1] for f in fs])
        hs = (C.c_int * n)(*[f.shape[0] for f in fs])
        ptrs = (C.c_void_p * n)(*[f.ctypes.data for f in fs])
        mptrs, keep_m = _mask_ptrs(masks, n)
        w, h = self.canvas[0], self.canvas[1]
        rgb = np.zeros((h, w, 3), np.uint8)
        mask = np.zeros((h, w), np.uint8)
        rep = RefReport()
        rc = lib().ref_process_sized(self._h, n, ws, hs, ptrs, mptrs, rgb.ctypes.data,
                                     mask.ctypes.data, C.byref(rep))
        if rc != OK:
            raise RefError(rc)
        return rgb, mask, rep

    def close(self):
        if self._h:
            lib().ref_state_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_curve(m1, m2, gamma_dark=1.5, gamma_bright=1.5, tb=0, tw=255) -> np.ndarray:
    """stitch::build_curve (color_balance.cpp:65-104) -> (3, 256) u8."""
    out = np.zeros((3, 256), np.uint8)
    lib().ref_build_curve((C.c_int * 3)(*m1), (C.c_int * 3)(*m2), gamma_dark, gamma_bright,
                          tb, tw, out.ctypes.data)
    return out


def _p(a):
    return None if a is None else np.ascontiguousarray(a, np.uint8).ctypes.data


def dense_flow(a_rgb, a_mask, b_rgb, b_mask, levels=4, iterations=50, smoothness=15.0,
               threads=1):
    """stitch::dense_flow (flow.cpp:140-187) -> (u, v) float32."""
    a_rgb, b_rgb = (np.ascontiguousarray(x, np.uint8) for x in (a_rgb, b_rgb))
    a_mask = None if a_mask is None else np.ascontiguousarray(a_mask, np.uint8)
    b_mask = None if b_mask is None else np.ascontiguousarray(b_mask, np.uint8)
    h, w = a_rgb.shape[:2]
    u = np.zeros((h, w), np.float32)
    v = np.zeros((h, w), np.float32)
    rc = lib().ref_dense_flow(w, h, _p(a_rgb), _p(a_mask), _p(b_rgb), _p(b_mask), levels,
                              iterations, smoothness, threads,
                              u.ctypes.data_as(C.POINTER(C.c_float)),
                              v.ctypes.data_as(C.POINTER(C.c_float)))
    if rc != OK:
        raise RefError(rc)
    return u, v


def warp_frame(rgb, mask, h9, cw, ch, ox, oy):
    """stitch::warp_frame (geometry.cpp:58-83) -> (rgb, mask) on the canvas."""
    rgb = np.ascontiguousarray(rgb, np.uint8)
    mask = None if mask is None else np.ascontiguousarray(mask, np.uint8)
    h, w = rgb.shape[:2]
    out = np.zeros((ch, cw, 3), np.uint8)
    om = np.zeros((ch, cw), np.uint8)
    hm = (C.c_double * 9)(*np.asarray(h9, np.float64).reshape(9))
    rc = lib().ref_warp_frame(w, h, _p(rgb), _p(mask), hm, cw, ch, ox, oy, out.ctypes.data,
                              om.ctypes.data)
    if rc != OK:
        raise RefError(rc)
    return out, om
