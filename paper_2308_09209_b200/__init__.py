"""B200-native per-frame video stitching (arXiv 2308.09209 hot path).

The compute path is libstitch_b200.so (hand-written sm_100a CUDA behind the
C ABI in include/stitch_b200.h).  This package is the host-side mirror of the
reference's pipeline API (proj/include/stitch/pipeline.hpp) over that ABI.
Importing it fails loudly when the shared library has not been built.
"""
from . import _abi
from .pipeline import (  # noqa: F401
    BalanceConfig,
    CameraExtrinsics,
    CameraIntrinsics,
    ErrorCode,
    FlickerEvent,
    FlowOptions,
    Frame,
    FrameReport,
    ParallaxObject,
    PipelineState,
    ProcessResult,
    RefineOptions,
    RunReport,
    RunResult,
    STAGE_NAMES,
    StitchConfig,
    StitchError,
    SynthScene,
    SynthSpec,
    ViewSetup,
    camera_maps,
    compare_methods,
    MetricRow,
    psnr,
    ssim,
    create_from_init,
    initialize,
    process_frame,
    run_sequence,
    read_ppm,
    write_ppm,
    read_png,
    write_png,
    read_image,
    write_image,
    sequence_name,
    list_sequence,
    run_files,
    FilesResult,
)

lib = _abi.load()
__version__ = lib.stitch_b200_version().decode()
