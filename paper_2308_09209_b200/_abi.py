"""ctypes declarations of include/stitch_b200.h (the C ABI of libstitch_b200.so)."""
from __future__ import annotations

import ctypes as C
import os

MAX_VIEWS = 16
MAX_PAIRS = 16

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libstitch_b200.so")
SYNTH_LIB_PATH = os.path.join(_HERE, "libstitch_synth.so")


class Camera(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("rotation", C.c_double * 9), ("translation", C.c_double * 3)]


class Config(C.Structure):
    _fields_ = [("n_views", C.c_int), ("reference", C.c_int),
                ("width", C.c_int * MAX_VIEWS), ("height", C.c_int * MAX_VIEWS),
                ("cams", Camera * MAX_VIEWS),
                ("lambda_", C.c_double), ("gamma_dark", C.c_double), ("gamma_bright", C.c_double),
                ("target_black", C.c_int), ("target_white", C.c_int),
                ("flow_levels", C.c_int), ("flow_iterations", C.c_int),
                ("smoothness", C.c_double), ("window_capacity", C.c_int),
                ("fuse_weighting", C.c_int), ("topology", C.c_int), ("refine_enabled", C.c_int),
                ("projection", C.c_int), ("cyl_focal", C.c_double),
                ("refine_margin", C.c_double), ("ransac_iters", C.c_int),
                ("inlier_px", C.c_double), ("detect_threshold", C.c_double),
                ("match_ratio", C.c_double), ("seed", C.c_ulonglong)]


class Pair(C.Structure):
    _fields_ = [("view", C.c_int), ("partner", C.c_int), ("x0", C.c_int), ("y0", C.c_int),
                ("x1", C.c_int), ("y1", C.c_int), ("theta_i", C.POINTER(C.c_float))]


class Init(C.Structure):
    _fields_ = [("canvas_width", C.c_int), ("canvas_height", C.c_int),
                ("canvas_offset", C.c_double * 2), ("n_views", C.c_int), ("reference", C.c_int),
                ("view_width", C.c_int * MAX_VIEWS), ("view_height", C.c_int * MAX_VIEWS),
                ("inv_maps", (C.c_double * 9) * MAX_VIEWS), ("n_pairs", C.c_int),
                ("pairs", Pair * MAX_PAIRS), ("window_capacity", C.c_int),
                ("lambda_", C.c_double), ("gamma_dark", C.c_double), ("gamma_bright", C.c_double),
                ("target_black", C.c_int), ("target_white", C.c_int),
                ("flow_levels", C.c_int), ("flow_iterations", C.c_int),
                ("smoothness", C.c_double), ("fuse_weighting", C.c_int),
                ("projection", C.c_int), ("cyl_focal", C.c_double)]


class Report(C.Structure):
    _fields_ = [("frame_index", C.c_longlong), ("n_pairs", C.c_int),
                ("color_matrices", (C.c_double * 9) * MAX_PAIRS),
                ("rank_deficient", C.c_int * MAX_PAIRS),
                ("threshold_m1", C.c_int * 3), ("threshold_m2", C.c_int * 3),
                ("balanced", C.c_int), ("stage_ms", C.c_double * 4)]


class Flicker(C.Structure):
    _fields_ = [("frame", C.c_int), ("view", C.c_int), ("gains", C.c_double * 3)]


class SynthSpec(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("views", C.c_int), ("frames", C.c_int),
                ("width", C.c_int), ("height", C.c_int), ("overlap_fraction", C.c_double),
                ("n_casts", C.c_int), ("color_casts", (C.c_double * 3) * MAX_VIEWS),
                ("n_flicker", C.c_int), ("flicker", Flicker * 16),
                ("object_enabled", C.c_int), ("object_depth_fraction", C.c_double),
                ("object_half_size", C.c_double), ("object_position", C.c_double * 2),
                ("object_velocity", C.c_double * 2), ("perturb_focal_scale", C.c_double),
                ("perturb_principal_px", C.c_double), ("rig", C.c_int),
                ("strip_yaw", C.c_double)]


class FilesStats(C.Structure):
    _fields_ = [("frames", C.c_longlong), ("seconds", C.c_double),
                ("read_seconds", C.c_double), ("write_seconds", C.c_double)]


# exported symbols (name, restype, argtypes) -- every declaration of the header
SYMBOLS = [
    ("stitch_b200_last_error", C.c_char_p, []),
    ("stitch_b200_version", C.c_char_p, []),
    ("stitch_b200_config_defaults", None, [C.POINTER(Config)]),
    ("stitch_b200_create", C.c_int, [C.POINTER(Init), C.c_int, C.POINTER(C.c_void_p)]),
    ("stitch_b200_initialize", C.c_int, [C.POINTER(Config), C.c_int, C.POINTER(C.c_void_p)]),
    ("stitch_b200_update_geometry", C.c_int, [C.c_void_p, C.POINTER(Init)]),
    ("stitch_b200_update_maps", C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    ("stitch_b200_initialize_frames_masked", C.c_int, [C.POINTER(Config), C.POINTER(C.c_void_p),
                                                       C.POINTER(C.c_void_p), C.c_int,
                                                       C.POINTER(C.c_void_p)]),
    ("stitch_b200_initialize_frames", C.c_int, [C.POINTER(Config), C.c_void_p, C.c_int,
                                                C.POINTER(C.c_void_p)]),
    ("stitch_b200_rerefine_masked", C.c_int, [C.c_void_p, C.POINTER(Config),
                                              C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    ("stitch_b200_refine_warning", C.c_int, [C.c_void_p, C.c_int]),
    ("stitch_b200_rerefine", C.c_int, [C.c_void_p, C.POINTER(Config), C.c_void_p]),
    ("stitch_b200_process_device_async", C.c_int, [C.c_void_p, C.c_void_p]),
    ("stitch_b200_fork", C.c_int, [C.c_void_p]),
    ("stitch_b200_join", C.c_int, [C.c_void_p]),
    ("stitch_b200_debug_detect", C.c_int, [C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_int),
                                           C.c_double, C.c_int, C.c_void_p, C.c_void_p]),
    ("stitch_b200_debug_match", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_double,
                                          C.c_void_p, C.c_void_p, C.c_void_p]),
    ("stitch_b200_debug_tone_curves", C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_double,
                                                C.c_double, C.c_int, C.c_int, C.c_void_p]),
    ("stitch_b200_camera_maps", C.c_int, [C.POINTER(Config), C.POINTER(C.c_double)]),
    ("stitch_b200_psnr", C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.POINTER(C.c_double)]),
    ("stitch_b200_ssim", C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.POINTER(C.c_double)]),
    ("stitch_b200_pair_quality", C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_double)]),
    ("stitch_b200_destroy", None, [C.c_void_p]),
    ("stitch_b200_canvas", C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                     C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("stitch_b200_n_pairs", C.c_int, [C.c_void_p]),
    ("stitch_b200_get_pair", C.c_int, [C.c_void_p, C.c_int, C.POINTER(Pair), C.c_void_p]),
    ("stitch_b200_view_bbox", C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int)]),
    ("stitch_b200_get_inv_map", C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_double)]),
    ("stitch_b200_process", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.c_void_p, C.c_void_p,
                                      C.POINTER(Report)]),
    ("stitch_b200_submit", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.c_void_p, C.c_void_p,
                                     C.POINTER(C.c_longlong)]),
    ("stitch_b200_wait", C.c_int, [C.c_void_p, C.c_longlong, C.POINTER(Report)]),
    ("stitch_b200_process_device", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p),
                                             C.POINTER(Report)]),
    ("stitch_b200_device_pano", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p),
                                          C.POINTER(C.c_void_p)]),
    ("stitch_b200_stream", C.c_void_p, [C.c_void_p]),
    ("stitch_b200_synchronize", C.c_int, [C.c_void_p]),
    ("stitch_b200_launches_per_frame", C.c_int, [C.c_void_p]),
    ("stitch_b200_profile_frame", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.c_int,
                                            C.POINTER(C.c_int), C.POINTER(C.c_float)]),
    ("stitch_b200_ppm_info", C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("stitch_b200_read_ppm", C.c_int, [C.c_char_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_int),
                                       C.POINTER(C.c_int)]),
    ("stitch_b200_write_ppm", C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_void_p]),
    ("stitch_b200_sequence_name", C.c_int, [C.c_char_p, C.c_int, C.c_char_p, C.c_char_p,
                                            C.c_size_t]),
    ("stitch_b200_run_files", C.c_int, [C.c_void_p, C.POINTER(C.c_char_p), C.c_char_p,
                                        C.c_char_p, C.c_char_p, C.c_int, C.c_void_p,
                                        C.POINTER(FilesStats)]),
    ("stitch_b200_read_png", C.c_int, [C.c_char_p, C.c_void_p, C.c_size_t, C.c_void_p,
                                       C.c_size_t, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                       C.POINTER(C.c_int)]),
    ("stitch_b200_write_png", C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    ("stitch_b200_n_views", C.c_int, [C.c_void_p]),
    ("stitch_b200_process_masked", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p),
                                             C.POINTER(C.c_void_p), C.c_void_p, C.c_void_p,
                                             C.c_void_p]),
    ("stitch_b200_submit_masked", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p),
                                            C.POINTER(C.c_void_p), C.c_void_p, C.c_void_p,
                                            C.POINTER(C.c_longlong)]),
    ("stitch_b200_slots", C.c_int, [C.c_void_p]),
    ("stitch_b200_check_frames", C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int),
                                           C.POINTER(C.c_int), C.c_void_p]),
    ("stitch_b200_view_size", C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int),
                                        C.POINTER(C.c_int)]),
    ("stitch_b200_set_error", C.c_int, [C.c_int, C.c_char_p]),
    ("stitch_b200_host_alloc", C.c_void_p, [C.c_size_t]),
    ("stitch_b200_host_free", None, [C.c_void_p]),
    ("stitch_b200_host_register", C.c_int, [C.c_void_p, C.c_size_t]),
    ("stitch_b200_debug_copy_pool", C.c_int, [C.c_int, C.c_int, C.c_size_t]),
    ("stitch_b200_host_unregister", C.c_int, [C.c_void_p]),
    ("stitch_b200_device_alloc", C.c_void_p, [C.c_int, C.c_size_t]),
    ("stitch_b200_device_free", None, [C.c_void_p]),
    ("stitch_b200_memcpy_h2d", C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t]),
    ("stitch_b200_memcpy_d2h", C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t]),
    ("stitch_b200_debug_crop", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                         C.c_void_p]),
    ("stitch_b200_debug_flow", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
    ("stitch_b200_debug_prebalance", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("stitch_b200_debug_warp_view", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                              C.c_void_p]),

]

OP_KIND_NAMES = ["expand_rgba", "crop_warp", "pair_color", "pair_solve", "flow_prepare", "pyr_down", "hs_linearize",
                 "hs_sweeps", "canvas_balance", "balance", "tone", "event"]

SYNTH_SYMBOLS = [
    ("stitch_b200_synth_defaults", None, [C.POINTER(SynthSpec)]),
    ("stitch_b200_synth_create", C.c_int, [C.POINTER(SynthSpec), C.POINTER(C.c_void_p)]),
    ("stitch_b200_synth_destroy", None, [C.c_void_p]),
    ("stitch_b200_synth_reference", C.c_int, [C.c_void_p]),
    ("stitch_b200_synth_config", C.c_int, [C.c_void_p, C.POINTER(Config)]),
    ("stitch_b200_synth_render", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int]),
]

_lib = None
_synth = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libstitch_b200.so; raises (never falls back) when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `make -C paper_2308_09209_b200` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(path)
    for name, restype, argtypes in SYMBOLS:
        fn = getattr(lib, name)
        fn.restype = restype
        fn.argtypes = argtypes
    _lib = lib
    return lib


def load_synth(path: str = SYNTH_LIB_PATH) -> C.CDLL:
    """Load libstitch_synth.so (the synthetic scene generator: test and bench
    inputs, include/stitch_synth.h) -- without the B200 product library."""
    global _synth
    if _synth is not None:
        return _synth
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `make -C paper_2308_09209_b200`")
    lib = C.CDLL(path)
    for name, restype, argtypes in SYNTH_SYMBOLS:
        fn = getattr(lib, name)
        fn.restype = restype
        fn.argtypes = argtypes
    _synth = lib
    return lib
