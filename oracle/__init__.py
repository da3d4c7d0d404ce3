"""CPU ORACLE -- test infrastructure only.

ctypes binding of oracle/liboracle.so, the plain-C restatement of the
reference's per-frame stitching path (see stitch_oracle.h for the citation
map and the parity status).  Only tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline / `--impl reference` legs may import this package,
and only as the checker or as the timed CPU baseline; the B200 product never
imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

MAX_VIEWS = 16
_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")

ERROR_NAMES = ["EmptyRegion", "EmptyHistogram", "RankDeficient", "RegionTooSmall",
               "InsufficientMatches", "NoConsensus", "ShapeMismatch", "NoOverlap",
               "SingularHomography", "DegeneratePose", "EmptyProjection", "MissingState",
               "TooSmall", "ConfigError", "ConfigurationError", "InputMismatch", "IoError"]
SO_OK = -1


class SoFrame(C.Structure):
    _fields_ = [("width", C.c_int), ("height", C.c_int), ("data", C.POINTER(C.c_uint8)),
                ("mask", C.POINTER(C.c_uint8))]


class SoRegion(C.Structure):
    _fields_ = [("x0", C.c_int), ("y0", C.c_int), ("x1", C.c_int), ("y1", C.c_int)]


class SoHist(C.Structure):
    _fields_ = [("bins", (C.c_uint32 * 256) * 3), ("total", C.c_uint64)]


class SoCamera(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("rotation", C.c_double * 9), ("translation", C.c_double * 3)]


class SoConfig(C.Structure):
    _fields_ = [("n_views", C.c_int), ("reference", C.c_int),
                ("width", C.c_int * MAX_VIEWS), ("height", C.c_int * MAX_VIEWS),
                ("cams", SoCamera * MAX_VIEWS),
                ("lambda_", C.c_double), ("gamma_dark", C.c_double), ("gamma_bright", C.c_double),
                ("target_black", C.c_int), ("target_white", C.c_int),
                ("flow_levels", C.c_int), ("flow_iterations", C.c_int),
                ("smoothness", C.c_double), ("window_capacity", C.c_int),
                ("fuse_weighting", C.c_int), ("topology", C.c_int), ("threads", C.c_int),
                ("keep_debug", C.c_int), ("projection", C.c_int), ("cyl_focal", C.c_double),
                ("refine_enabled", C.c_int), ("refine_margin", C.c_double),
                ("ransac_iters", C.c_int), ("inlier_px", C.c_double),
                ("detect_threshold", C.c_double), ("match_ratio", C.c_double),
                ("seed", C.c_ulonglong)]


class SoKeypoint(C.Structure):
    _fields_ = [("x", C.c_double), ("y", C.c_double), ("scale", C.c_double),
                ("response", C.c_double)]


class SoMatchPair(C.Structure):
    _fields_ = [("index_a", C.c_int), ("index_b", C.c_int), ("distance", C.c_double),
                ("ax", C.c_double), ("ay", C.c_double), ("bx", C.c_double), ("by", C.c_double)]


class SoSimilarity(C.Structure):
    _fields_ = [("s_x", C.c_double), ("s_y", C.c_double), ("t_x", C.c_double),
                ("t_y", C.c_double)]


class SoReport(C.Structure):
    _fields_ = [("frame_index", C.c_long), ("n_pairs", C.c_int),
                ("m", (C.c_double * 9) * MAX_VIEWS), ("rank_deficient", C.c_int * MAX_VIEWS),
                ("threshold_m1", C.c_int * 3), ("threshold_m2", C.c_int * 3),
                ("balanced", C.c_int), ("stage_seconds", C.c_double * 4)]


_lib = None


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc, no FMA)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return LIB_PATH


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        build()
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    sigs = {
        "so_quantize_channel": (C.c_uint8, [C.c_double]),
        "so_sample_bilinear": (C.c_int, [P(SoFrame), C.c_double, C.c_double, P(C.c_float)]),
        "so_compute_histogram": (C.c_int, [P(SoFrame), SoRegion, P(SoHist)]),
        "so_cdf": (C.c_int, [P(SoHist), C.c_void_p]),
        "so_inverse3": (None, [P(C.c_double), P(C.c_double)]),
        "so_det3": (C.c_double, [P(C.c_double)]),
        "so_warp_frame": (C.c_int, [P(SoFrame), P(C.c_double), C.c_int, C.c_int, C.c_double,
                                    C.c_double, C.c_int, P(SoFrame)]),
        "so_histogram_specification": (C.c_int, [P(SoHist), P(SoHist), C.c_void_p]),
        "so_solve_color_matrix": (C.c_int, [C.c_int, P(C.c_int), P(C.c_void_p), P(C.c_void_p),
                                            P(C.c_double), P(C.c_double)]),
        "so_sym3_eigen": (None, [P(C.c_double), P(C.c_double)]),
        "so_ldlt_solve3": (None, [P(C.c_double), P(C.c_double), P(C.c_double)]),
        "so_apply_color_matrix_rows": (None, [P(SoFrame), P(C.c_double), C.c_int]),
        "so_find_thresholds": (C.c_int, [P(SoHist), C.c_double, P(C.c_int), P(C.c_int)]),
        "so_smooth_thresholds": (None, [C.c_int, C.c_void_p, C.c_void_p, P(C.c_int),
                                        P(C.c_int)]),
        "so_balance_curve_value": (C.c_double, [C.c_double, C.c_int, C.c_int, C.c_double,
                                                C.c_double, C.c_int, C.c_int]),
        "so_build_curve": (C.c_int, [P(C.c_int), P(C.c_int), C.c_double, C.c_double, C.c_int,
                                     C.c_int, C.c_void_p]),
        "so_dense_flow": (C.c_int, [P(SoFrame), P(SoFrame), C.c_int, C.c_int, C.c_double,
                                    C.c_int, P(C.c_float), P(C.c_float)]),
        "so_blend_weights": (None, [P(SoFrame), P(SoFrame), SoRegion, P(C.c_float),
                                    P(C.c_float)]),
        "so_flow_fuse": (C.c_int, [P(SoFrame), P(SoFrame)] + [P(C.c_float)] * 6 +
                         [C.c_int, P(SoFrame)]),
        "so_compose_panorama": (C.c_int, [P(SoFrame), P(SoFrame), P(SoFrame), SoRegion,
                                          P(SoFrame)]),
        "so_initialize": (C.c_void_p, [P(SoConfig), P(C.c_int)]),
        "so_destroy": (None, [C.c_void_p]),
        "so_process_frame": (C.c_int, [C.c_void_p, P(SoFrame), P(SoFrame), P(SoReport)]),
        "so_state_canvas": (None, [C.c_void_p, P(C.c_int), P(C.c_int), P(C.c_double),
                                   P(C.c_double)]),
        "so_state_map": (None, [C.c_void_p, C.c_int, P(C.c_double), P(C.c_double)]),
        "so_state_n_pairs": (C.c_int, [C.c_void_p]),
        "so_state_pair": (None, [C.c_void_p, C.c_int, P(C.c_int), P(C.c_int), P(SoRegion)]),
        "so_state_pair_weights": (None, [C.c_void_p, C.c_int, P(C.c_float)]),
        "so_state_view_bbox": (None, [C.c_void_p, C.c_int, P(SoRegion)]),
        "so_state_last_flow": (C.c_int, [C.c_void_p, C.c_int, C.c_int, P(C.c_float),
                                         P(C.c_float)]),
        "so_state_last_warped": (C.c_int, [C.c_void_p, C.c_int, P(C.c_uint8), P(C.c_uint8)]),
        "so_free_frame": (None, [P(SoFrame)]),
        "so_psnr": (C.c_int, [P(SoFrame), P(SoFrame), P(C.c_double)]),
        "so_detect": (C.c_int, [P(SoFrame), SoRegion, C.c_double, P(P(SoKeypoint)), P(C.c_int)]),
        "so_describe": (None, [P(SoFrame), P(SoKeypoint), C.c_int, P(C.c_float)]),
        "so_match": (C.c_int, [P(C.c_float), C.c_int, P(C.c_float), C.c_int, P(SoKeypoint),
                               P(SoKeypoint), C.c_double, P(SoMatchPair)]),
        "so_ransac": (C.c_int, [P(SoMatchPair), C.c_int, C.c_int, C.c_double, C.c_double,
                                C.c_double, C.c_ulonglong, P(SoSimilarity)]),
        "so_initialize_frames": (C.c_void_p, [P(SoConfig), P(SoFrame), P(C.c_int)]),
        "so_state_refine_warning": (C.c_int, [C.c_void_p, C.c_int]),
        "so_ssim": (C.c_int, [P(SoFrame), P(SoFrame), P(C.c_double)]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


class OracleError(RuntimeError):
    def __init__(self, code: int):
        self.code = code
        super().__init__(ERROR_NAMES[code] if 0 <= code < len(ERROR_NAMES) else f"code {code}")


# ---------------------------------------------------------------------------
# numpy <-> so_frame
# ---------------------------------------------------------------------------
class FrameRef:
    """Keeps numpy buffers alive behind an SoFrame."""

    def __init__(self, data: np.ndarray, mask=None):
        self.data = np.ascontiguousarray(data, dtype=np.uint8)
        self.mask = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        h, w = self.data.shape[:2]
        self.c = SoFrame(w, h, self.data.ctypes.data_as(C.POINTER(C.c_uint8)),
                         None if self.mask is None else
                         self.mask.ctypes.data_as(C.POINTER(C.c_uint8)))


def take_frame(f: SoFrame):
    """Copy an oracle-allocated frame into numpy and free it."""
    h, w = f.height, f.width
    data = np.ctypeslib.as_array(f.data, shape=(h * w * 3,)).copy().reshape(h, w, 3)
    mask = None
    if f.mask:
        mask = np.ctypeslib.as_array(f.mask, shape=(h * w,)).copy().reshape(h, w)
    lib().so_free_frame(C.byref(f))
    return data, mask


def psnr(a_data, a_mask, b_data, b_mask) -> float:
    """metrics.cpp:9-31 (oracle)."""
    fa, fb = FrameRef(a_data, a_mask), FrameRef(b_data, b_mask)
    out = C.c_double()
    e = lib().so_psnr(C.byref(fa.c), C.byref(fb.c), C.byref(out))
    if e != SO_OK:
        raise OracleError(e)
    return out.value


def ssim(a_data, a_mask, b_data, b_mask) -> float:
    """metrics.cpp:83-155 (oracle)."""
    fa, fb = FrameRef(a_data, a_mask), FrameRef(b_data, b_mask)
    out = C.c_double()
    e = lib().so_ssim(C.byref(fa.c), C.byref(fb.c), C.byref(out))
    if e != SO_OK:
        raise OracleError(e)
    return out.value


def detect(data, mask, region, threshold=2e-4):
    """features.cpp:52-118 -> list of (x, y, scale, response)."""
    fr = FrameRef(data, mask)
    out = C.POINTER(SoKeypoint)()
    n = C.c_int()
    e = lib().so_detect(C.byref(fr.c), SoRegion(*region), threshold, C.byref(out), C.byref(n))
    if e != SO_OK:
        raise OracleError(e)
    kps = [(out[i].x, out[i].y, out[i].scale, out[i].response) for i in range(n.value)]
    if n.value:
        C.CDLL(None).free(out)
    return kps


def _kp_array(kps):
    arr = (SoKeypoint * max(1, len(kps)))()
    for i, k in enumerate(kps):
        arr[i] = SoKeypoint(*k)
    return arr


def describe(data, mask, kps):
    """features.cpp:139-179 -> (n, 64) float32."""
    fr = FrameRef(data, mask)
    out = np.zeros((max(1, len(kps)), 64), np.float32)
    lib().so_describe(C.byref(fr.c), _kp_array(kps), len(kps),
                      out.ctypes.data_as(C.POINTER(C.c_float)))
    return out[:len(kps)]


def match(da, db, ka, kb, ratio=0.8):
    """features.cpp:181-234 -> list of (a, b, distance, ax, ay, bx, by)."""
    da = np.ascontiguousarray(da, np.float32)
    db = np.ascontiguousarray(db, np.float32)
    out = (SoMatchPair * max(1, len(ka)))()
    n = lib().so_match(da.ctypes.data_as(C.POINTER(C.c_float)), len(ka),
                       db.ctypes.data_as(C.POINTER(C.c_float)), len(kb), _kp_array(ka),
                       _kp_array(kb), ratio, out)
    return [(out[i].index_a, out[i].index_b, out[i].distance, out[i].ax, out[i].ay, out[i].bx,
             out[i].by) for i in range(n)]


def ransac(matches, iterations=500, inlier_px=2.0, min_scale=0.5, max_scale=2.0, seed=0):
    """features.cpp:282-354 on (ax, ay, bx, by[, distance]) -> (s_x, s_y, t_x, t_y)."""
    arr = (SoMatchPair * max(1, len(matches)))()
    for i, m in enumerate(matches):
        ax, ay, bx, by = m[:4]
        d = m[4] if len(m) > 4 else 0.0
        arr[i] = SoMatchPair(i, i, d, ax, ay, bx, by)
    out = SoSimilarity()
    e = lib().so_ransac(arr, len(matches), iterations, inlier_px, min_scale, max_scale, seed,
                        C.byref(out))
    if e != SO_OK:
        raise OracleError(e)
    return (out.s_x, out.s_y, out.t_x, out.t_y)


def quantize_channel(v: float) -> int:
    return int(lib().so_quantize_channel(v))


def sample_bilinear(data, mask, x: float, y: float):
    fr = FrameRef(data, mask)
    out = (C.c_float * 3)()
    ok = lib().so_sample_bilinear(C.byref(fr.c), x, y, out)
    return bool(ok), np.array(out[:], dtype=np.float32)


def compute_histogram(data, mask, region):
    fr = FrameRef(data, mask)
    h = SoHist()
    rc = lib().so_compute_histogram(C.byref(fr.c), SoRegion(*region), C.byref(h))
    if rc != SO_OK:
        raise OracleError(rc)
    return np.array([h.bins[c][:] for c in range(3)], dtype=np.uint64), int(h.total)


def _hist(bins, total=None) -> SoHist:
    h = SoHist()
    bins = np.asarray(bins)
    for c in range(3):
        for v in range(256):
            h.bins[c][v] = int(bins[c][v])
    h.total = int(bins[0].sum()) if total is None else int(total)
    return h


def cdf(bins, total=None):
    h = _hist(bins, total)
    out = (C.c_double * (3 * 256))()
    rc = lib().so_cdf(C.byref(h), out)
    if rc != SO_OK:
        raise OracleError(rc)
    return np.array(out[:]).reshape(3, 256)


def histogram_specification(src_bins, ref_bins):
    hs, hr = _hist(src_bins), _hist(ref_bins)
    out = (C.c_uint8 * 768)()
    rc = lib().so_histogram_specification(C.byref(hs), C.byref(hr), out)
    if rc != SO_OK:
        raise OracleError(rc)
    return np.array(out[:], dtype=np.uint8).reshape(3, 256)


def solve_color_matrix(window):
    """window: list of (src_rows n x 3, tgt_rows n x 3), newest first."""
    n = len(window)
    rows = (C.c_int * max(1, n))(*[len(s) for s, _ in window])
    keep = [(np.ascontiguousarray(s, np.float64), np.ascontiguousarray(t, np.float64))
            for s, t in window]
    sp = (C.c_void_p * max(1, n))(*[s.ctypes.data for s, _ in keep])
    tp = (C.c_void_p * max(1, n))(*[t.ctypes.data for _, t in keep])
    m = (C.c_double * 9)()
    sv = C.c_double(0)
    rc = lib().so_solve_color_matrix(n, rows, sp, tp, m, C.byref(sv))
    if rc != SO_OK:
        raise OracleError(rc)
    return np.array(m[:]).reshape(3, 3), sv.value


def apply_color_matrix_rows(data, mask, m):
    fr = FrameRef(np.array(data, copy=True), mask)
    mm = (C.c_double * 9)(*np.asarray(m, np.float64).reshape(9))
    lib().so_apply_color_matrix_rows(C.byref(fr.c), mm, 1)
    return fr.data


def find_thresholds(bins, lam, total=None):
    h = _hist(bins, total)
    m1, m2 = (C.c_int * 3)(), (C.c_int * 3)()
    rc = lib().so_find_thresholds(C.byref(h), lam, m1, m2)
    if rc != SO_OK:
        raise OracleError(rc)
    return list(m1), list(m2)


def smooth_thresholds(history):
    """history: list of (m1[3], m2[3]) newest last."""
    n = len(history)
    a1 = (C.c_int * (3 * max(1, n)))(*[v for h in history for v in h[0]])
    a2 = (C.c_int * (3 * max(1, n)))(*[v for h in history for v in h[1]])
    o1, o2 = (C.c_int * 3)(), (C.c_int * 3)()
    lib().so_smooth_thresholds(n, a1, a2, o1, o2)
    return list(o1), list(o2)


def build_curve(m1, m2, gamma_dark=1.5, gamma_bright=1.5, tb=0, tw=255):
    out = (C.c_uint8 * 768)()
    rc = lib().so_build_curve((C.c_int * 3)(*m1), (C.c_int * 3)(*m2), gamma_dark, gamma_bright,
                              tb, tw, out)
    if rc != SO_OK:
        raise OracleError(rc)
    return np.array(out[:], dtype=np.uint8).reshape(3, 256)


def warp_frame(data, inv, cw, ch, offx, offy, threads=1):
    fr = FrameRef(data)
    out = SoFrame()
    invc = (C.c_double * 9)(*np.asarray(inv, np.float64).reshape(9))
    rc = lib().so_warp_frame(C.byref(fr.c), invc, cw, ch, offx, offy, threads, C.byref(out))
    if rc != SO_OK:
        lib().so_free_frame(C.byref(out))
        raise OracleError(rc)
    return take_frame(out)


def dense_flow(a_data, a_mask, b_data, b_mask, levels=4, iterations=50, smoothness=15.0,
               threads=1):
    fa, fb = FrameRef(a_data, a_mask), FrameRef(b_data, b_mask)
    h, w = fa.data.shape[:2]
    u = np.zeros((h, w), np.float32)
    v = np.zeros((h, w), np.float32)
    rc = lib().so_dense_flow(C.byref(fa.c), C.byref(fb.c), levels, iterations, smoothness,
                             threads, u.ctypes.data_as(C.POINTER(C.c_float)),
                             v.ctypes.data_as(C.POINTER(C.c_float)))
    if rc != SO_OK:
        raise OracleError(rc)
    return u, v


def flow_fuse(ri, rj, uij, vij, uji, vji, theta_i, theta_j=None, weighting=0):
    fi, fj = FrameRef(*ri), FrameRef(*rj)
    if theta_j is None:
        theta_j = (np.float32(1.0) - np.asarray(theta_i, np.float32)).astype(np.float32)
    arrs = [np.ascontiguousarray(a, np.float32) for a in (uij, vij, uji, vji, theta_i, theta_j)]
    ptrs = [a.ctypes.data_as(C.POINTER(C.c_float)) for a in arrs]
    out = SoFrame()
    rc = lib().so_flow_fuse(C.byref(fi.c), C.byref(fj.c), *ptrs, weighting, C.byref(out))
    if rc != SO_OK:
        raise OracleError(rc)
    return take_frame(out)


def compose_panorama(wi, wj, fused, region):
    a, b, f = FrameRef(*wi), FrameRef(*wj), FrameRef(*fused)
    out = SoFrame()
    rc = lib().so_compose_panorama(C.byref(a.c), C.byref(b.c), C.byref(f.c), SoRegion(*region),
                                   C.byref(out))
    if rc != SO_OK:
        raise OracleError(rc)
    return take_frame(out)


def blend_weights(mask_i, mask_j, region):
    h, w = mask_i.shape
    zi = np.zeros((h, w, 3), np.uint8)
    fi, fj = FrameRef(zi, mask_i), FrameRef(zi, mask_j)
    bw, bh = region[2] - region[0], region[3] - region[1]
    ti = np.zeros((bh, bw), np.float32)
    tj = np.zeros((bh, bw), np.float32)
    lib().so_blend_weights(C.byref(fi.c), C.byref(fj.c), SoRegion(*region),
                           ti.ctypes.data_as(C.POINTER(C.c_float)),
                           tj.ctypes.data_as(C.POINTER(C.c_float)))
    return ti, tj


# ---------------------------------------------------------------------------
# pipeline
# ---------------------------------------------------------------------------
def make_config(n_views, reference, sizes, cams, *, lam=0.05, gamma_dark=1.5, gamma_bright=1.5,
                target_black=0, target_white=255, levels=4, iterations=50, smoothness=15.0,
                window=3, weighting=0, topology=0, threads=1, keep_debug=0, projection=0,
                cyl_focal=0.0, refine=False, refine_margin=0.15, ransac_iters=500,
                inlier_px=2.0, detect_threshold=2e-4, match_ratio=0.8, seed=0) -> SoConfig:
    """cams: list of (fx, fy, cx, cy, R[9] row-major, t[3])."""
    c = SoConfig()
    c.n_views = n_views
    c.reference = reference
    for v in range(n_views):
        c.width[v], c.height[v] = sizes[v]
        fx, fy, cx, cy, r, t = cams[v]
        c.cams[v].fx, c.cams[v].fy, c.cams[v].cx, c.cams[v].cy = fx, fy, cx, cy
        for i in range(9):
            c.cams[v].rotation[i] = float(r[i])
        for i in range(3):
            c.cams[v].translation[i] = float(t[i])
    c.lambda_ = lam
    c.gamma_dark, c.gamma_bright = gamma_dark, gamma_bright
    c.target_black, c.target_white = target_black, target_white
    c.flow_levels, c.flow_iterations, c.smoothness = levels, iterations, smoothness
    c.window_capacity = window
    c.fuse_weighting = weighting
    c.topology = topology
    c.threads = threads
    c.keep_debug = keep_debug
    c.projection = projection
    c.cyl_focal = cyl_focal
    c.refine_enabled = 1 if refine else 0
    c.refine_margin, c.ransac_iters, c.inlier_px = refine_margin, ransac_iters, inlier_px
    c.detect_threshold, c.match_ratio, c.seed = detect_threshold, match_ratio, seed
    return c


class OracleState:
    """so_state: the oracle's PipelineState (initialize + process_frame)."""

    def __init__(self, cfg: SoConfig, first_frames=None, first_masks=None):
        self.cfg = cfg
        err = C.c_int(SO_OK)
        if first_frames is not None:
            fm = first_masks or [None] * len(first_frames)
            refs = [FrameRef(f, m) for f, m in zip(first_frames, fm)]
            arr = (SoFrame * len(refs))(*[r.c for r in refs])
            self._h = lib().so_initialize_frames(C.byref(cfg), arr, C.byref(err))
        else:
            self._h = lib().so_initialize(C.byref(cfg), C.byref(err))
        if not self._h:
            raise OracleError(err.value)
        w, h, ox, oy = C.c_int(), C.c_int(), C.c_double(), C.c_double()
        lib().so_state_canvas(self._h, C.byref(w), C.byref(h), C.byref(ox), C.byref(oy))
        self.canvas = (w.value, h.value, ox.value, oy.value)

    def n_pairs(self) -> int:
        return lib().so_state_n_pairs(self._h)

    def pair(self, k):
        v, p, r = C.c_int(), C.c_int(), SoRegion()
        lib().so_state_pair(self._h, k, C.byref(v), C.byref(p), C.byref(r))
        return v.value, p.value, (r.x0, r.y0, r.x1, r.y1)

    def pair_weights(self, k):
        _, _, b = self.pair(k)
        out = np.zeros((b[3] - b[1], b[2] - b[0]), np.float32)
        lib().so_state_pair_weights(self._h, k, out.ctypes.data_as(C.POINTER(C.c_float)))
        return out

    def view_bbox(self, v):
        r = SoRegion()
        lib().so_state_view_bbox(self._h, v, C.byref(r))
        return (r.x0, r.y0, r.x1, r.y1)

    def refine_warning(self, k) -> bool:
        return bool(lib().so_state_refine_warning(self._h, k))

    def maps(self, v):
        h = (C.c_double * 9)()
        inv = (C.c_double * 9)()
        lib().so_state_map(self._h, v, h, inv)
        return np.array(h[:]).reshape(3, 3), np.array(inv[:]).reshape(3, 3)

    def process(self, frames, masks=None):
        """frames: RGB8 arrays; masks: per frame None or an (H, W) 0/1 array
        (Frame::mask, frame.hpp:44-47)."""
        refs = [FrameRef(f, m) for f, m in zip(frames, masks or [None] * len(frames))]
        arr = (SoFrame * len(refs))(*[r.c for r in refs])
        out = SoFrame()
        rep = SoReport()
        rc = lib().so_process_frame(self._h, arr, C.byref(out), C.byref(rep))
        if rc != SO_OK:
            raise OracleError(rc)
        data, mask = take_frame(out)
        return data, mask, rep

    def last_flow(self, k, d):
        _, _, b = self.pair(k)
        shape = (b[3] - b[1], b[2] - b[0])
        u = np.zeros(shape, np.float32)
        v = np.zeros(shape, np.float32)
        rc = lib().so_state_last_flow(self._h, k, d, u.ctypes.data_as(C.POINTER(C.c_float)),
                                      v.ctypes.data_as(C.POINTER(C.c_float)))
        if rc != SO_OK:
            raise OracleError(rc)
        return u, v

    def last_warped(self, v):
        w, h = self.canvas[0], self.canvas[1]
        rgb = np.zeros((h, w, 3), np.uint8)
        mask = np.zeros((h, w), np.uint8)
        rc = lib().so_state_last_warped(self._h, v, rgb.ctypes.data_as(C.POINTER(C.c_uint8)),
                                        mask.ctypes.data_as(C.POINTER(C.c_uint8)))
        if rc != SO_OK:
            raise OracleError(rc)
        return rgb, mask

    def close(self):
        if self._h:
            lib().so_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
