"""Python mirror of the reference's pipeline API over the B200 C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/stitch/pipeline.hpp:17-92 (StitchConfig,
PipelineState, initialize, process_frame, run_sequence),
report.hpp:11-58 (Stage, FrameReport, RunReport) and types.hpp:9-44
(ErrorCode, StitchError).  Every frame goes through libstitch_b200.so; there
is no CPU path.
"""
from __future__ import annotations

import copy
import ctypes as C
import enum
import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _abi


class ErrorCode(enum.IntEnum):
    """stitch::ErrorCode (types.hpp:9-27)."""
    EmptyRegion = 0
    EmptyHistogram = 1
    RankDeficient = 2
    RegionTooSmall = 3
    InsufficientMatches = 4
    NoConsensus = 5
    ShapeMismatch = 6
    NoOverlap = 7
    SingularHomography = 8
    DegeneratePose = 9
    EmptyProjection = 10
    MissingState = 11
    TooSmall = 12
    ConfigError = 13
    ConfigurationError = 14
    InputMismatch = 15
    IoError = 16


class StitchError(RuntimeError):
    """stitch::StitchError (types.hpp:33-44); `code` is an ErrorCode, or None
    for device/runtime failures (status >= 100)."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status
        self.code = ErrorCode(status - 1) if 1 <= status <= 17 else None


def _lib():
    return _abi.load()


def _synth_lib():
    return _abi.load_synth()


def _check_synth(status: int) -> None:
    """status of a synthetic-scene call (libstitch_synth.so: codes only)."""
    if status != 0:
        raise StitchError(status, f"synthetic scene: status {status} "
                                  f"({ErrorCode(status - 1).name if 1 <= status <= 17 else '?'})")


def check(status: int) -> None:
    if status != 0:
        msg = _lib().stitch_b200_last_error().decode(errors="replace")
        raise StitchError(status, msg or f"stitch_b200 status {status}")


# ---------------------------------------------------------------------------
# Frames and config (frame.hpp:17-57, geometry.hpp:11-30, pipeline.hpp:17-44)
# ---------------------------------------------------------------------------
@dataclass
class Frame:
    """RGB8 raster (H, W, 3) with an optional 0/1 mask (H, W); None = all valid."""
    data: np.ndarray
    mask: Optional[np.ndarray] = None

    @property
    def width(self) -> int:
        return int(self.data.shape[1])

    @property
    def height(self) -> int:
        return int(self.data.shape[0])

    def has_mask(self) -> bool:
        return self.mask is not None


@dataclass
class CameraIntrinsics:
    fx: float = 1.0
    fy: float = 1.0
    cx: float = 0.0
    cy: float = 0.0


@dataclass
class CameraExtrinsics:
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))


@dataclass
class ViewSetup:
    intrinsics: CameraIntrinsics = field(default_factory=CameraIntrinsics)
    extrinsics: CameraExtrinsics = field(default_factory=CameraExtrinsics)
    dir: str = ""


@dataclass
class BalanceConfig:  # color_balance.hpp:19-25
    lambda_: float = 0.05
    gamma_dark: float = 1.5
    gamma_bright: float = 1.5
    target_black: int = 0
    target_white: int = 255


@dataclass
class FlowOptions:  # flow.hpp:29-34
    levels: int = 4
    iterations: int = 50
    smoothness: float = 15.0
    threads: int = 1


@dataclass
class RefineOptions:  # pipeline.hpp:23-31
    # Feature refinement runs at initialize() (detect / describe / match on
    # the device, RANSAC on the host), on by default like the reference.
    enabled: bool = True
    margin: float = 0.15
    ransac_iters: int = 500
    inlier_px: float = 2.0
    detect_threshold: float = 2e-4
    match_ratio: float = 0.8
    rerefine_every: int = 0


@dataclass
class StitchConfig:  # pipeline.hpp:33-44
    views: List[ViewSetup] = field(default_factory=list)
    reference: int = 0
    balance: BalanceConfig = field(default_factory=BalanceConfig)
    flow: FlowOptions = field(default_factory=FlowOptions)
    refine: RefineOptions = field(default_factory=RefineOptions)
    threads: int = 1
    seed: int = 0
    window_capacity: int = 3
    fuse_weighting: str = "own"  # "own" | "cross"
    scene_id: str = "scene"
    topology: str = "auto"  # extension: "auto" | "star" | "chain" | "ring"
    device: int = 0
    projection: str = "planar"  # extension: "planar" | "cylindrical" (360-degree rigs)
    cyl_focal: float = 0.0


def _config_to_c(cfg: StitchConfig, sizes: Sequence[tuple]) -> _abi.Config:
    c = _abi.Config()
    _lib().stitch_b200_config_defaults(C.byref(c))
    c.n_views = len(cfg.views)
    c.reference = cfg.reference
    for v, (setup, (w, h)) in enumerate(zip(cfg.views, sizes)):
        c.width[v] = int(w)
        c.height[v] = int(h)
        cam = c.cams[v]
        cam.fx, cam.fy = setup.intrinsics.fx, setup.intrinsics.fy
        cam.cx, cam.cy = setup.intrinsics.cx, setup.intrinsics.cy
        r = np.asarray(setup.extrinsics.rotation, dtype=np.float64).reshape(9)
        t = np.asarray(setup.extrinsics.translation, dtype=np.float64).reshape(3)
        for i in range(9):
            cam.rotation[i] = float(r[i])
        for i in range(3):
            cam.translation[i] = float(t[i])
    c.lambda_ = cfg.balance.lambda_
    c.gamma_dark = cfg.balance.gamma_dark
    c.gamma_bright = cfg.balance.gamma_bright
    c.target_black = cfg.balance.target_black
    c.target_white = cfg.balance.target_white
    c.flow_levels = cfg.flow.levels
    c.flow_iterations = cfg.flow.iterations
    c.smoothness = cfg.flow.smoothness
    c.window_capacity = cfg.window_capacity
    c.fuse_weighting = 1 if cfg.fuse_weighting == "cross" else 0
    c.topology = {"auto": 0, "star": 1, "chain": 2, "ring": 3}[cfg.topology]
    c.projection = 1 if cfg.projection == "cylindrical" else 0
    c.cyl_focal = cfg.cyl_focal
    c.refine_enabled = 1 if cfg.refine.enabled else 0
    c.refine_margin = cfg.refine.margin
    c.ransac_iters = cfg.refine.ransac_iters
    c.inlier_px = cfg.refine.inlier_px
    c.detect_threshold = cfg.refine.detect_threshold
    c.match_ratio = cfg.refine.match_ratio
    c.seed = int(cfg.seed) & 0xFFFFFFFFFFFFFFFF
    return c


def _config_from_c(c: _abi.Config) -> StitchConfig:
    cfg = StitchConfig(reference=c.reference)
    cfg.projection = "cylindrical" if c.projection == 1 else "planar"
    cfg.cyl_focal = c.cyl_focal
    cfg.topology = {0: "auto", 1: "star", 2: "chain", 3: "ring"}[c.topology]
    for v in range(c.n_views):
        cam = c.cams[v]
        cfg.views.append(ViewSetup(
            CameraIntrinsics(cam.fx, cam.fy, cam.cx, cam.cy),
            CameraExtrinsics(np.array(cam.rotation[:], dtype=np.float64).reshape(3, 3),
                             np.array(cam.translation[:], dtype=np.float64))))
    return cfg


# ---------------------------------------------------------------------------
# Report (report.hpp:11-58)
# ---------------------------------------------------------------------------
STAGE_NAMES = ("Geometric Warping", "Color Correction", "Local Warping", "Image Blending")


@dataclass
class FrameReport:
    frame_index: int = 0
    times: List[float] = field(default_factory=lambda: [0.0] * 4)  # seconds per Stage
    color_matrices: List[np.ndarray] = field(default_factory=list)
    rank_deficient: List[bool] = field(default_factory=list)
    threshold_m1: List[int] = field(default_factory=lambda: [0, 0, 0])
    threshold_m2: List[int] = field(default_factory=lambda: [0, 0, 0])
    balanced: bool = False


@dataclass
class RunReport:
    scene_id: str = ""
    threads: int = 1
    frames: int = 0
    totals: List[float] = field(default_factory=lambda: [0.0] * 4)
    wall_seconds: float = 0.0
    per_frame: List[FrameReport] = field(default_factory=list)
    refine_warning: bool = False

    def fps(self) -> float:
        return self.frames / self.wall_seconds if self.wall_seconds > 0 else 0.0


def _report_from_c(r: _abi.Report) -> FrameReport:
    out = FrameReport(frame_index=int(r.frame_index))
    out.times = [r.stage_ms[i] * 1e-3 for i in range(4)]
    for k in range(r.n_pairs):
        out.color_matrices.append(np.array(r.color_matrices[k][:], dtype=np.float64).reshape(3, 3))
        out.rank_deficient.append(bool(r.rank_deficient[k]))
    out.threshold_m1 = list(r.threshold_m1)
    out.threshold_m2 = list(r.threshold_m2)
    out.balanced = bool(r.balanced)
    return out


# ---------------------------------------------------------------------------
# Device context == PipelineState (pipeline.hpp:47-63)
# ---------------------------------------------------------------------------
@dataclass
class PairState:
    view: int
    partner: int
    bounds: tuple  # (x0, y0, x1, y1)
    theta_i: np.ndarray
    refine_warning: bool = False  # refinement fell back to the unrefined map


class PipelineState:
    """Owns one stitch_b200_ctx: the device-resident pipeline state of one
    panorama stream (canvas, maps, pairs, 3D-M windows, threshold history)."""

    def __init__(self, handle: C.c_void_p, config: Optional[StitchConfig] = None):
        self._h = handle
        self.config = config
        self._refresh()
        self.n_views = len(config.views) if config else None
        self.frame_counter = 0

    def _refresh(self) -> None:
        lib = _lib()
        w, h = C.c_int(), C.c_int()
        ox, oy = C.c_double(), C.c_double()
        check(lib.stitch_b200_canvas(self._h, C.byref(w), C.byref(h), C.byref(ox), C.byref(oy)))
        self.canvas = (w.value, h.value, ox.value, oy.value)
        self.pairs: List[PairState] = []
        for k in range(lib.stitch_b200_n_pairs(self._h)):
            p = _abi.Pair()
            check(lib.stitch_b200_get_pair(self._h, k, C.byref(p), None))
            th = np.empty((p.y1 - p.y0, p.x1 - p.x0), dtype=np.float32)
            check(lib.stitch_b200_get_pair(self._h, k, C.byref(p), th.ctypes.data_as(C.c_void_p)))
            self.pairs.append(PairState(p.view, p.partner, (p.x0, p.y0, p.x1, p.y1), th))

    def pair_quality(self, k: int) -> tuple:
        """Tables 2-3 columns of pair k in the last frame (device):
        (psnr(corrected, source), psnr(corrected, reference),
        ssim(corrected, reference))."""
        out = (C.c_double * 3)()
        check(_lib().stitch_b200_pair_quality(self._h, k, out))
        return tuple(out)

    def rerefine(self, config: StitchConfig, frames: Sequence[Frame]) -> None:
        """run_sequence's re-refinement (pipeline.cpp:395-406): a fresh
        initialize() on `frames` with the temporal state carried over."""
        c = _config_to_c(config, [(f.width, f.height) for f in frames])
        arrs, ptrs = _frame_ptrs(frames, len(config.views))
        if any(f.mask is not None for f in frames):
            keep, mptrs = _mask_ptrs(frames)
            check(_lib().stitch_b200_rerefine_masked(self._h, C.byref(c), ptrs, mptrs))
        else:
            check(_lib().stitch_b200_rerefine(self._h, C.byref(c), ptrs))
        self._refresh()
        for k, p in enumerate(self.pairs):
            p.refine_warning = bool(_lib().stitch_b200_refine_warning(self._h, k))

    def update_maps(self, maps: np.ndarray) -> None:
        """Re-refinement from new view->reference homographies (n, 3, 3):
        canvas, inverse maps and pair geometry rebuilt (the pair geometry on
        the device); windows, threshold history and counter carried over
        (pipeline.cpp:395-406)."""
        m = np.ascontiguousarray(maps, dtype=np.float64).reshape(-1)
        check(_lib().stitch_b200_update_maps(self._h, m.ctypes.data_as(C.POINTER(C.c_double))))
        self._refresh()

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    @property
    def canvas_width(self) -> int:
        return self.canvas[0]

    @property
    def canvas_height(self) -> int:
        return self.canvas[1]

    def view_bbox(self, view: int) -> tuple:
        b = (C.c_int * 4)()
        check(_lib().stitch_b200_view_bbox(self._h, view, b))
        return tuple(b)

    def inv_map(self, view: int) -> np.ndarray:
        m = (C.c_double * 9)()
        check(_lib().stitch_b200_get_inv_map(self._h, view, m))
        return np.array(m[:], dtype=np.float64).reshape(3, 3)

    def launches_per_frame(self) -> int:
        return _lib().stitch_b200_launches_per_frame(self._h)

    def close(self) -> None:
        if self._h:
            _lib().stitch_b200_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class ProcessResult:  # pipeline.hpp:65-68
    panorama: Frame
    report: FrameReport


def initialize(config: StitchConfig, first_frames: Sequence[Frame]) -> PipelineState:
    """pipeline.hpp:73-74; with refine.enabled (the default, as in the
    reference) the first frames feed the feature refinement, and masked first
    frames (Frame.mask) the pair geometry."""
    if len(first_frames) != len(config.views):
        raise StitchError(ErrorCode.ConfigurationError + 1,
                          "frame count does not match configured views")
    sizes = [(f.width, f.height) for f in first_frames]
    c = _config_to_c(config, sizes)
    h = C.c_void_p()
    if any(f.mask is not None for f in first_frames):
        # masked first frames decide the pair geometry (pipeline.cpp:181-205)
        arrs, ptrs = _frame_ptrs(first_frames, len(config.views))
        keep, mptrs = _mask_ptrs(first_frames)
        check(_lib().stitch_b200_initialize_frames_masked(C.byref(c), ptrs, mptrs, config.device,
                                                          C.byref(h)))
    elif config.refine.enabled:
        arrs, ptrs = _frame_ptrs(first_frames, len(config.views))
        check(_lib().stitch_b200_initialize_frames(C.byref(c), ptrs, config.device, C.byref(h)))
    else:
        check(_lib().stitch_b200_initialize(C.byref(c), config.device, C.byref(h)))
    state = PipelineState(h, config)
    for k, p in enumerate(state.pairs):
        p.refine_warning = bool(_lib().stitch_b200_refine_warning(h, k))
    return state


def camera_maps(config: StitchConfig, sizes: Sequence[tuple]) -> np.ndarray:
    """The unrefined view->reference homographies initialize() derives from
    the camera models (pipeline.cpp:219-229), shape (n, 3, 3)."""
    c = _config_to_c(config, sizes)
    out = np.zeros((len(config.views), 3, 3), dtype=np.float64)
    check(_lib().stitch_b200_camera_maps(C.byref(c), out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def _metric(fn, a: Frame, b: Frame) -> float:
    if a.data.shape != b.data.shape:
        raise StitchError(ErrorCode.ShapeMismatch + 1, "frame sizes differ")
    da = np.ascontiguousarray(a.data, np.uint8)
    db = np.ascontiguousarray(b.data, np.uint8)
    ma = None if a.mask is None else np.ascontiguousarray(a.mask, np.uint8)
    mb = None if b.mask is None else np.ascontiguousarray(b.mask, np.uint8)
    out = C.c_double()
    check(fn(a.width, a.height, da.ctypes.data, None if ma is None else ma.ctypes.data,
             db.ctypes.data, None if mb is None else mb.ctypes.data, C.byref(out)))
    return out.value


def psnr(a: Frame, b: Frame) -> float:
    """metrics.hpp:15 psnr(a, b), evaluated on the device."""
    return _metric(_lib().stitch_b200_psnr, a, b)


def ssim(a: Frame, b: Frame) -> float:
    """metrics.hpp:21 ssim(a, b), evaluated on the device."""
    return _metric(_lib().stitch_b200_ssim, a, b)


@dataclass
class MetricRow:  # metrics.hpp:23-30
    scene_id: str
    frame_label: str
    method: str
    psnr_vs_source: float = 0.0
    psnr_vs_reference: float = 0.0
    ssim_vs_reference: float = 0.0


def compare_methods(config: StitchConfig, views: Sequence[Sequence[Frame]], pair: int = 0,
                    scene_id: str = "") -> List[MetricRow]:
    """The Tables 2-3 comparison (metrics.hpp:48-54, compare_methods_both) on
    the stitching pipeline's own overlap of `pair`: the sequence runs once
    with window 1 (2D-M) and once with window 3 (3D-M); per-frame rows then
    mu and sigma (population) rows per method."""
    rows: List[MetricRow] = []
    for window, method in ((1, "2D-M"), (3, "3D-M")):
        cfg = copy.deepcopy(config)
        cfg.window_capacity = window
        state = initialize(cfg, [s[0] for s in views])
        cols = []
        try:
            for t in range(len(views[0])):
                process_frame(state, [s[t] for s in views])
                q = state.pair_quality(pair)
                rows.append(MetricRow(scene_id, str(t + 1), method, *q))
                cols.append(q)
        finally:
            state.close()
        arr = np.array(cols, dtype=np.float64)
        mu = arr.mean(axis=0)
        sigma = np.sqrt(((arr - mu) ** 2).mean(axis=0))
        rows.append(MetricRow(scene_id, "mu", method, *mu))
        rows.append(MetricRow(scene_id, "sigma", method, *sigma))
    return rows


def create_from_init(init: _abi.Init, device: int = 0,
                     config: Optional[StitchConfig] = None) -> PipelineState:
    """Drop-in path: a state snapshot produced elsewhere (e.g. the reference's
    own initialize() with feature refinement) -> device context."""
    h = C.c_void_p()
    check(_lib().stitch_b200_create(C.byref(init), device, C.byref(h)))
    return PipelineState(h, config)


def _frame_ptrs(frames: Sequence[Frame], n: int):
    if len(frames) != n:
        raise StitchError(ErrorCode.ConfigurationError + 1,
                          "frame count does not match configured views")
    arrs = []
    for f in frames:
        a = np.ascontiguousarray(f.data, dtype=np.uint8)
        if a.ndim != 3 or a.shape[2] != 3:
            raise StitchError(ErrorCode.InputMismatch + 1, "frames must be (H, W, 3) uint8")
        if f.mask is not None and np.asarray(f.mask).shape != a.shape[:2]:
            raise StitchError(ErrorCode.InputMismatch + 1, "frame mask must be (H, W)")
        arrs.append(a)
    ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    return arrs, ptrs


def _mask_ptrs(frames: Sequence[Frame]):
    masks = [None if f.mask is None else np.ascontiguousarray(f.mask, dtype=np.uint8)
             for f in frames]
    ptrs = (C.c_void_p * len(masks))(*[None if m is None else m.ctypes.data for m in masks])
    return masks, ptrs


def check_frames(state: PipelineState, frames: Sequence[Frame]) -> None:
    """stitch_b200_check_frames: frame count and per-view size as initialized
    -- InputMismatch instead of a silent misread."""
    n = len(frames)
    ws = (C.c_int * max(1, n))(*[f.width for f in frames])
    hs = (C.c_int * max(1, n))(*[f.height for f in frames])
    keep, mptrs = _mask_ptrs(frames)
    check(_lib().stitch_b200_check_frames(state.handle, n, ws, hs, mptrs))


def process_frame(state: PipelineState, frames: Sequence[Frame]) -> ProcessResult:
    """pipeline.hpp:79-80: one frame through warp -> 3D-M colour -> flow ->
    blend -> balance, on the GPU."""
    n = len(state.config.views) if state.config else len(frames)
    arrs, ptrs = _frame_ptrs(frames, n)
    check_frames(state, frames)
    w, h = state.canvas_width, state.canvas_height
    rgb = np.empty((h, w, 3), dtype=np.uint8)
    mask = np.empty((h, w), dtype=np.uint8)
    rep = _abi.Report()
    if any(f.mask is not None for f in frames):
        # masked inputs (Frame::mask): the sampler skips masked taps (frame.cpp:95-104)
        keep, mptrs = _mask_ptrs(frames)
        check(_lib().stitch_b200_process_masked(state.handle, ptrs, mptrs,
                                                rgb.ctypes.data_as(C.c_void_p),
                                                mask.ctypes.data_as(C.c_void_p), C.byref(rep)))
    else:
        check(_lib().stitch_b200_process(state.handle, ptrs, rgb.ctypes.data_as(C.c_void_p),
                                         mask.ctypes.data_as(C.c_void_p), C.byref(rep)))
    state.frame_counter += 1
    return ProcessResult(Frame(rgb, mask), _report_from_c(rep))


@dataclass
class RunResult:
    panoramas: List[Frame]
    report: RunReport


def run_sequence(config: StitchConfig, views: Sequence[Sequence[Frame]],
                 sink: Optional[Callable[[int, Frame], None]] = None) -> RunResult:
    """pipeline.hpp:90-92 / pipeline.cpp:362-420, including the re-refinement
    branch (refine.rerefine_every > 0)."""
    if len(views) != len(config.views):
        raise StitchError(ErrorCode.ConfigurationError + 1,
                          "stream count does not match configured views")
    frames = len(views[0])
    if any(len(s) != frames for s in views):
        raise StitchError(ErrorCode.ConfigurationError + 1, "streams must have equal length")
    if frames == 0:
        raise StitchError(ErrorCode.ConfigurationError + 1, "empty input streams")
    t0 = time.perf_counter()
    state = initialize(config, [s[0] for s in views])
    result = RunResult([], RunReport(scene_id=config.scene_id, threads=config.threads,
                                     frames=frames))
    # pipeline.cpp:390-392: any pair whose refinement fell back
    result.report.refine_warning = any(p.refine_warning for p in state.pairs)
    try:
        every = config.refine.rerefine_every
        for t in range(frames):
            if every > 0 and t > 0 and t % every == 0:
                state.rerefine(config, [s[t] for s in views])
            pr = process_frame(state, [s[t] for s in views])
            for i in range(4):
                result.report.totals[i] += pr.report.times[i]
            result.report.per_frame.append(pr.report)
            if sink:
                sink(t, pr.panorama)
            else:
                result.panoramas.append(pr.panorama)
    finally:
        state.close()
    result.report.wall_seconds = time.perf_counter() - t0
    return result


# ---------------------------------------------------------------------------
# Frame ingress / egress (image_io.hpp / image_io.cpp:19-199)
# ---------------------------------------------------------------------------
def read_ppm(path) -> Frame:
    """read_ppm (image_io.cpp:61-76): P6, maxval 255; IoError otherwise."""
    lib = _lib()
    p = str(path).encode()
    w, h = C.c_int(), C.c_int()
    check(lib.stitch_b200_read_ppm(p, None, 0, C.byref(w), C.byref(h)))
    data = np.empty((h.value, w.value, 3), np.uint8)
    check(lib.stitch_b200_read_ppm(p, data.ctypes.data_as(C.c_void_p), data.nbytes, None, None))
    return Frame(data)


def write_ppm(path, frame: Frame) -> None:
    """write_ppm (image_io.cpp:78-85); the mask is not stored (PPM is RGB)."""
    data = np.ascontiguousarray(frame.data, dtype=np.uint8)
    check(_lib().stitch_b200_write_ppm(str(path).encode(), frame.width, frame.height,
                                       data.ctypes.data_as(C.c_void_p)))


def read_png(path) -> Frame:
    """read_png (image_io.cpp:87-129): 8-bit RGB after libpng's expand /
    strip_16 / gray_to_rgb; transparent pixels become the mask (None when
    every pixel is opaque)."""
    lib = _lib()
    p = str(path).encode()
    w, h, hm = C.c_int(), C.c_int(), C.c_int()
    check(lib.stitch_b200_read_png(p, None, 0, None, 0, C.byref(w), C.byref(h), C.byref(hm)))
    data = np.empty((h.value, w.value, 3), np.uint8)
    mask = np.empty((h.value, w.value), np.uint8)
    check(lib.stitch_b200_read_png(p, data.ctypes.data_as(C.c_void_p), data.nbytes,
                                   mask.ctypes.data_as(C.c_void_p), mask.nbytes, None, None, None))
    return Frame(data, mask if hm.value else None)


def write_png(path, frame: Frame) -> None:
    """write_png (image_io.cpp:131-165): RGB, or RGBA with the mask as alpha."""
    data = np.ascontiguousarray(frame.data, dtype=np.uint8)
    mask = None if frame.mask is None else np.ascontiguousarray(frame.mask, dtype=np.uint8)
    check(_lib().stitch_b200_write_png(str(path).encode(), frame.width, frame.height,
                                       data.ctypes.data_as(C.c_void_p),
                                       None if mask is None else mask.ctypes.data_as(C.c_void_p)))


def read_image(path) -> Frame:
    """read_image (image_io.cpp:167-172): dispatch on .ppm / .png."""
    import os

    ext = os.path.splitext(str(path))[1]
    if ext == ".ppm":
        return read_ppm(path)
    if ext == ".png":
        return read_png(path)
    raise StitchError(ErrorCode.IoError + 1, f"{path}: unsupported image extension")


def write_image(path, frame: Frame) -> None:
    """write_image (image_io.cpp:174-179)."""
    import os

    ext = os.path.splitext(str(path))[1]
    if ext == ".ppm":
        return write_ppm(path, frame)
    if ext == ".png":
        return write_png(path, frame)
    raise StitchError(ErrorCode.IoError + 1, f"{path}: unsupported image extension")


def sequence_name(stem: str, index: int, ext: str = ".png") -> str:
    """sequence_name (image_io.cpp:194-199): stem_000003.png."""
    buf = C.create_string_buffer(len(stem) + len(ext) + 32)
    check(_lib().stitch_b200_sequence_name(stem.encode(), index, ext.encode(), buf, len(buf)))
    return buf.value.decode()


def list_sequence(directory) -> List[str]:
    """list_sequence (image_io.cpp:181-192): the .png / .ppm regular files of
    a directory, sorted by name; IoError when it is not a directory."""
    import os

    d = str(directory)
    if not os.path.isdir(d):
        raise StitchError(ErrorCode.IoError + 1, f"{d}: not a directory")
    return sorted(os.path.join(d, f) for f in os.listdir(d)
                  if os.path.isfile(os.path.join(d, f)) and os.path.splitext(f)[1] in (".png", ".ppm"))


@dataclass
class FilesResult:
    reports: List[FrameReport]
    frames: int
    seconds: float
    read_seconds: float
    write_seconds: float

    def fps(self) -> float:
        return self.frames / self.seconds if self.seconds > 0 else 0.0


def run_files(state: PipelineState, view_dirs: Sequence[str], out_dir: Optional[str] = None,
              stem: str = "pano", max_frames: int = 0, ext: str = ".ppm") -> FilesResult:
    """run_sequence (pipeline.cpp:364-412) on numbered .ppm / .png
    sequences, one directory per view, panoramas written as
    out_dir/stem_%06d<ext> (.ppm, or .png with the mask as alpha); file reads,
    the pipelined GPU frames and the writes overlap (C++ threads in
    libstitch_b200.so)."""
    lib = _lib()
    n = lib.stitch_b200_n_views(state.handle)
    if len(view_dirs) != n:
        raise StitchError(ErrorCode.InputMismatch + 1, "one directory per view")
    dirs = (C.c_char_p * n)(*[str(d).encode() for d in view_dirs])
    cap = max_frames if max_frames > 0 else min(len(list_sequence(d)) for d in view_dirs)
    reps = (_abi.Report * max(1, cap))()
    st = _abi.FilesStats()
    check(lib.stitch_b200_run_files(state.handle, dirs, str(out_dir).encode() if out_dir else None,
                                    stem.encode(), ext.encode(), cap, reps, C.byref(st)))
    return FilesResult([_report_from_c(reps[i]) for i in range(st.frames)], st.frames,
                       st.seconds, st.read_seconds, st.write_seconds)


# ---------------------------------------------------------------------------
# Synthetic scenes (synth.hpp:17-87)
# ---------------------------------------------------------------------------
@dataclass
class FlickerEvent:
    frame: int = 0
    view: int = 0
    gains: tuple = (1.0, 1.0, 1.0)


@dataclass
class ParallaxObject:
    enabled: bool = False
    depth_fraction: float = 0.15
    half_size: float = 40.0
    position: tuple = (0.0, 0.0)
    velocity: tuple = (0.0, 0.0)


@dataclass
class SynthSpec:
    seed: int = 1
    views: int = 2
    frames: int = 5
    width: int = 320
    height: int = 240
    overlap_fraction: float = 0.3
    color_casts: List[tuple] = field(default_factory=list)
    flicker: List[FlickerEvent] = field(default_factory=list)
    object: ParallaxObject = field(default_factory=ParallaxObject)
    perturb_focal_scale: float = 1.0
    perturb_principal_px: float = 0.0
    rig: str = "auto"  # "auto" | "yaw" (reference) | "strip" | "ring" (N-view extensions)
    strip_yaw: float = 0.05

    def to_c(self) -> _abi.SynthSpec:
        s = _abi.SynthSpec()
        _synth_lib().stitch_b200_synth_defaults(C.byref(s))
        s.seed = self.seed
        s.views = self.views
        s.frames = self.frames
        s.width = self.width
        s.height = self.height
        s.overlap_fraction = self.overlap_fraction
        s.n_casts = len(self.color_casts)
        for v, g in enumerate(self.color_casts):
            for c in range(3):
                s.color_casts[v][c] = float(g[c])
        s.n_flicker = len(self.flicker)
        for i, f in enumerate(self.flicker):
            s.flicker[i].frame = f.frame
            s.flicker[i].view = f.view
            for c in range(3):
                s.flicker[i].gains[c] = float(f.gains[c])
        s.object_enabled = 1 if self.object.enabled else 0
        s.object_depth_fraction = self.object.depth_fraction
        s.object_half_size = self.object.half_size
        s.object_position[0], s.object_position[1] = self.object.position
        s.object_velocity[0], s.object_velocity[1] = self.object.velocity
        s.perturb_focal_scale = self.perturb_focal_scale
        s.perturb_principal_px = self.perturb_principal_px
        s.rig = {"auto": 0, "yaw": 1, "strip": 2, "ring": 3}[self.rig]
        s.strip_yaw = self.strip_yaw
        return s


class SynthScene:
    """synth.hpp:49-87: procedural plane scene + cameras + renderer."""

    def __init__(self, spec: SynthSpec):
        self.spec = spec
        self._c = spec.to_c()
        self._h = C.c_void_p()
        _check_synth(_synth_lib().stitch_b200_synth_create(C.byref(self._c), C.byref(self._h)))

    def reference_view(self) -> int:
        return _synth_lib().stitch_b200_synth_reference(self._h)

    def config_c(self) -> _abi.Config:
        c = _abi.Config()
        _check_synth(_synth_lib().stitch_b200_synth_config(self._h, C.byref(c)))
        return c

    def config(self) -> StitchConfig:
        cfg = _config_from_c(self.config_c())
        cfg.seed = self.spec.seed
        cfg.scene_id = f"synth-{self.spec.seed}"
        # feature refinement (on by default, like the reference) serves the
        # planar canvas; the 360-degree ring extension keeps its exact maps
        if cfg.projection == "cylindrical":
            cfg.refine.enabled = False
        return cfg

    def render_view(self, view: int, frame: int, threads: int = 0) -> Frame:
        out = np.empty((self.spec.height, self.spec.width, 3), dtype=np.uint8)
        _check_synth(_synth_lib().stitch_b200_synth_render(self._h, view, frame,
                                              out.ctypes.data_as(C.c_void_p), threads))
        return Frame(out, None)

    def render_streams(self, frames: Optional[int] = None, threads: int = 0) -> List[List[Frame]]:
        n = self.spec.frames if frames is None else frames
        return [[self.render_view(v, t, threads) for t in range(n)] for v in range(self.spec.views)]

    def close(self):
        if self._h:
            _synth_lib().stitch_b200_synth_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
