/*
 * stitch_b200.h -- C ABI of the B200-native per-frame stitching path.
 *
 * Drop-in boundary for the reference's
 *   ProcessResult stitch::process_frame(PipelineState&, const std::vector<Frame>&)
 *   (/root/reference/proj/include/stitch/pipeline.hpp:79-80,
 *    impl proj/src/pipeline.cpp:259-360).
 * A context (stitch_b200_ctx) is the device-resident twin of one
 * PipelineState (pipeline.hpp:47-63): canvas, per-view inverse maps, pairs
 * {view, bounds, blend weights, 3D-M window}, threshold history, frame
 * counter.  One context per panorama stream; not thread-shared.
 *
 * Plain C types only; no exceptions cross this boundary.  Every entry point
 * returns STITCH_B200_OK (0) or a positive code mirroring stitch::ErrorCode
 * (proj/include/stitch/types.hpp:9-27) offset by 1; the message of the last
 * failure on the calling thread is available from stitch_b200_last_error().
 */
#ifndef STITCH_B200_H
#define STITCH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STITCH_B200_MAX_VIEWS 16
#define STITCH_B200_MAX_PAIRS 16

/* Return codes: 0 = OK, else 1 + stitch::ErrorCode (types.hpp:9-27),
 * plus codes >= 100 for device/runtime failures. */
enum stitch_b200_status {
  STITCH_B200_OK = 0,
  STITCH_B200_EmptyRegion = 1,
  STITCH_B200_EmptyHistogram = 2,
  STITCH_B200_RankDeficient = 3,
  STITCH_B200_RegionTooSmall = 4,
  STITCH_B200_InsufficientMatches = 5,
  STITCH_B200_NoConsensus = 6,
  STITCH_B200_ShapeMismatch = 7,
  STITCH_B200_NoOverlap = 8,
  STITCH_B200_SingularHomography = 9,
  STITCH_B200_DegeneratePose = 10,
  STITCH_B200_EmptyProjection = 11,
  STITCH_B200_MissingState = 12,
  STITCH_B200_TooSmall = 13,
  STITCH_B200_ConfigError = 14,
  STITCH_B200_ConfigurationError = 15,
  STITCH_B200_InputMismatch = 16,
  STITCH_B200_IoError = 17,
  STITCH_B200_CudaError = 100,
  STITCH_B200_Unsupported = 101
};

/* CameraIntrinsics + CameraExtrinsics (geometry.hpp:11-30). */
typedef struct {
  double fx, fy, cx, cy;
  double rotation[9]; /* row-major, world -> camera */
  double translation[3];
} stitch_b200_camera;

/* StitchConfig (pipeline.hpp:33-44).  Feature refinement (refine_enabled,
 * RefineOptions pipeline.hpp:23-31) runs in stitch_b200_initialize_frames,
 * which receives the first frames it needs (planar canvas only). */
typedef struct {
  int n_views;
  int reference;
  int width[STITCH_B200_MAX_VIEWS];
  int height[STITCH_B200_MAX_VIEWS];
  stitch_b200_camera cams[STITCH_B200_MAX_VIEWS];
  /* BalanceConfig, color_balance.hpp:19-25 */
  double lambda;
  double gamma_dark, gamma_bright;
  int target_black, target_white;
  /* FlowOptions, flow.hpp:29-34 */
  int flow_levels, flow_iterations;
  double smoothness;
  int window_capacity; /* 1..3 (clamped like TransferWindow) */
  int fuse_weighting;  /* 0 = own (OwnWeightOnOwnFlow), 1 = cross */
  int topology;        /* 0 = auto (star <= 3 views, chain beyond), 1 star, 2 chain,
                          3 ring chain (360 degree rigs) */
  int refine_enabled;  /* 1: refine_pair at init (stitch_b200_initialize_frames) */
  /* Extension (not in the reference, which is planar only): 0 = planar
   * canvas (the reference's world plane), 1 = cylindrical 360-degree canvas
   * around the reference camera, cyl_focal pixels per radian (0: the
   * reference camera's fx).  Cameras must share their centre. */
  int projection;
  double cyl_focal;
  /* RefineOptions (pipeline.hpp:23-31) and StitchConfig.seed */
  double refine_margin;     /* 0.15 */
  int ransac_iters;         /* 500 */
  double inlier_px;         /* 2.0 */
  double detect_threshold;  /* 2e-4 */
  double match_ratio;       /* 0.8 */
  unsigned long long seed;  /* RANSAC seed base (+ view index) */
} stitch_b200_config;

/* Fill a config with the reference defaults (pipeline.hpp:23-44,
 * color_balance.hpp:19-25, flow.hpp:29-34), feature refinement included
 * (refine_enabled = 1, pipeline.hpp:24: initialize with the first frames,
 * stitch_b200_initialize_frames). */
void stitch_b200_config_defaults(stitch_b200_config* cfg);

/* POD snapshot of an initialised PipelineState: the exact values the
 * reference's process_frame reads (pipeline.cpp:259-360). */
typedef struct {
  int view;    /* PairState::view */
  int partner; /* reference view (star) or neighbour (chain extension) */
  int x0, y0, x1, y1;    /* PairState::bounds (types.hpp:47-62) */
  const float* theta_i;  /* PairState::weights.theta_i, (y1-y0)*(x1-x0), row-major */
} stitch_b200_pair;

typedef struct {
  int canvas_width, canvas_height; /* CanvasGeometry (geometry.hpp:87-91) */
  double canvas_offset[2];
  int n_views, reference;
  int view_width[STITCH_B200_MAX_VIEWS];
  int view_height[STITCH_B200_MAX_VIEWS];
  /* warp_maps[v].h.inverse() exactly as pipeline.cpp:40 computes it (raw
   * Eigen cofactor inverse, not renormalised), row-major. */
  double inv_maps[STITCH_B200_MAX_VIEWS][9];
  int n_pairs;
  stitch_b200_pair pairs[STITCH_B200_MAX_PAIRS];
  /* StitchConfig fields read per frame */
  int window_capacity;
  double lambda, gamma_dark, gamma_bright;
  int target_black, target_white;
  int flow_levels, flow_iterations;
  double smoothness;
  int fuse_weighting;
  /* 0: planar -- inv_maps are the inverse homographies applied to
   * (x + offset_x, y + offset_y, 1).  1: cylindrical extension -- inv_maps
   * are K_v R_v R_ref^T applied to (sin t, h, cos t) with
   * t = (x + offset_x) / cyl_focal, h = (y + offset_y) / cyl_focal; a
   * sample is valid only in front of the camera. */
  int projection;
  double cyl_focal;
} stitch_b200_init;

/* FrameReport (report.hpp:38-45) without the host-only fields. */
typedef struct {
  long long frame_index;
  int n_pairs;
  double color_matrices[STITCH_B200_MAX_PAIRS][9]; /* row-major M per pair */
  int rank_deficient[STITCH_B200_MAX_PAIRS];
  int threshold_m1[3], threshold_m2[3];
  int balanced; /* 0 when the panorama histogram was empty */
  /* Stage::{GeometricWarping, ColorCorrection, LocalWarping, ImageBlending}
   * (report.hpp:11-17): device milliseconds between CUDA events recorded at
   * the stage boundaries of this frame's slot.  With several frames in
   * flight these are wall intervals on a GPU shared with the other frames'
   * kernels (and include waits on the previous frame's colour solve /
   * canvas), not the stage's exclusive cost the reference's
   * FrameReport.times measures on one thread; the per-kernel cost of a frame
   * run alone is what stitch_b200_profile_frame reports. */
  double stage_ms[4];
} stitch_b200_report;

typedef struct stitch_b200_ctx stitch_b200_ctx;

const char* stitch_b200_last_error(void);
const char* stitch_b200_version(void);

/* Create a device context from a state snapshot (reference-side
 * initialize() output).  Copies everything it needs. */
int stitch_b200_create(const stitch_b200_init* init, int device,
                       stitch_b200_ctx** out);

/* Standalone initialize (pipeline.cpp:209-257 with refinement off): camera
 * homographies and canvas on the host; warp masks, view footprints, overlap
 * bounds and chamfer blend weights (rebuild_pair_geometry,
 * pipeline.cpp:181-205) on the device. */
int stitch_b200_initialize(const stitch_b200_config* cfg, int device,
                           stitch_b200_ctx** out);

/* initialize() with the first frames (host RGB8, one per view): with
 * cfg->refine_enabled the maps are refined from feature matches on the
 * warped first frames (refine_pair, pipeline.cpp:114-179: detection,
 * description and matching on the device, RANSAC on the host with the
 * reference's std::mt19937_64 stream), then the pair geometry is rebuilt on
 * the device (pipeline.cpp:241-255). */
int stitch_b200_initialize_frames(const stitch_b200_config* cfg,
                                  const uint8_t* const* frames, int device,
                                  stitch_b200_ctx** out);
/* initialize_frames with masked first frames (masks: NULL, or per view NULL /
 * width*height bytes, 0 = invalid): the pair bounds and blend weights follow
 * the masked warps of the first frames, as the reference's
 * rebuild_pair_geometry warps first_frames (pipeline.cpp:181-205); the
 * feature refinement warps them with the masked sampler too.  A masked first
 * frame without one valid warped pixel is STITCH_B200_EmptyProjection
 * (checked before the overlaps, as the reference warps every view first). */
int stitch_b200_initialize_frames_masked(const stitch_b200_config* cfg,
                                         const uint8_t* const* frames,
                                         const uint8_t* const* masks, int device,
                                         stitch_b200_ctx** out);

/* run_sequence's re-refinement branch (pipeline.cpp:395-406): a fresh
 * initialize(config, current frames) (with refinement when enabled) replaces
 * the context's geometry; the 3D-M windows, threshold history and frame
 * counter are carried over.  The pair set must not change. */
int stitch_b200_rerefine(stitch_b200_ctx* ctx, const stitch_b200_config* cfg,
                         const uint8_t* const* frames);
/* rerefine with the current frames' masks (NULL, or per view NULL / W*H
 * bytes): run_sequence's re-initialize on masked frames. */
int stitch_b200_rerefine_masked(stitch_b200_ctx* ctx, const stitch_b200_config* cfg,
                                const uint8_t* const* frames, const uint8_t* const* masks);

/* 1 when pair k's refinement fell back to the unrefined map
 * (PairState::refine_warning: too few keypoints / matches, no consensus). */
int stitch_b200_refine_warning(const stitch_b200_ctx* ctx, int k);

/* Re-upload geometry (re-refinement, pipeline.cpp:395-406): the 3D-M
 * windows, threshold history and frame counter are kept. */
int stitch_b200_update_geometry(stitch_b200_ctx* ctx,
                                const stitch_b200_init* init);

/* Re-refinement from new view->reference homographies (the refined
 * `warp_maps[v].h`, row-major, planar canvas only): the canvas
 * (compute_canvas, geometry.cpp:147-171), the inverse maps and the whole pair
 * geometry (rebuild_pair_geometry, pipeline.cpp:181-205) are recomputed --
 * the pair geometry on the device -- and the windows, threshold history and
 * frame counter are carried over as run_sequence does (pipeline.cpp:395-406).
 * The pair set is kept. */
int stitch_b200_update_maps(stitch_b200_ctx* ctx, const double* maps /* n_views * 9 */);

/* The unrefined view->reference homographies initialize() derives from the
 * camera models (pipeline.cpp:219-229), row-major, n_views * 9 doubles. */
int stitch_b200_camera_maps(const stitch_b200_config* cfg, double* maps);

void stitch_b200_destroy(stitch_b200_ctx* ctx);

/* Quality metrics (metrics.cpp:9-155), evaluated on the device, results
 * equal to the reference's.  psnr: dB over jointly valid pixels, channels
 * pooled, +inf for identical inputs; ssim: mean SSIM on Rec.601 luma with an
 * 11x11 Gaussian window (sigma 1.5) over windows with fully valid support.
 * Host RGB8 frames, masks 0/1 or NULL (all valid).  Errors: ShapeMismatch
 * is impossible here (one size), EmptyRegion, TooSmall (ssim, < 11 px). */
int stitch_b200_psnr(int width, int height, const uint8_t* a_rgb, const uint8_t* a_mask,
                     const uint8_t* b_rgb, const uint8_t* b_mask, double* out);
int stitch_b200_ssim(int width, int height, const uint8_t* a_rgb, const uint8_t* a_mask,
                     const uint8_t* b_rgb, const uint8_t* b_mask, double* out);

/* The paper's Tables 2-3 columns for pair k's colour transfer in the last
 * processed frame, on the device-resident overlap crops (compare_methods,
 * metrics.cpp:177-208, with the context's window capacity = the method):
 * out[0] = psnr(corrected, source), out[1] = psnr(corrected, reference),
 * out[2] = ssim(corrected, reference). */
int stitch_b200_pair_quality(stitch_b200_ctx* ctx, int k, double out[3]);

/* Feature-path diagnostics (the device kernels of stitch_b200_initialize_frames
 * on one host RGB8 frame, for parity tests): detect over region
 * {x0, y0, x1, y1} + describe; kp gets 4 doubles (x, y, scale, response) and
 * desc 64 floats per keypoint, at most max_kp.  Returns the keypoint count,
 * or minus an error code.  debug_match: the device matching of two
 * descriptor sets (best_b[a] = ratio-tested nearest b or -1, best_a[b]). */
int stitch_b200_debug_detect(int width, int height, const uint8_t* rgb, const int region[4],
                             double threshold, int max_kp, double* kp, float* desc);
/* Test entry: the device tone curve (build_curve, color_balance.cpp:65-104)
 * for n threshold pairs (m1[i], m2[i]) -> out[n * 256]. */
int stitch_b200_debug_tone_curves(int n, const int* m1, const int* m2, double gamma_dark,
                                  double gamma_bright, int target_black, int target_white,
                                  uint8_t* out);
int stitch_b200_debug_match(const float* da, int na, const float* db, int nb, double ratio,
                            int* best_b, double* best_dist, int* best_a);

/* Geometry of a context. */
int stitch_b200_canvas(const stitch_b200_ctx* ctx, int* width, int* height,
                       double* offset_x, double* offset_y);
int stitch_b200_n_pairs(const stitch_b200_ctx* ctx);
int stitch_b200_get_pair(const stitch_b200_ctx* ctx, int k,
                         stitch_b200_pair* pair, float* theta_i_out);
int stitch_b200_view_bbox(const stitch_b200_ctx* ctx, int view, int bbox[4]);
int stitch_b200_get_inv_map(const stitch_b200_ctx* ctx, int view,
                            double inv[9]);

/* One frame through the stage order (pipeline.cpp:259-360).
 * frames[v]: host RGB8 (width*height*3), pinned or pageable.  Outputs:
 * pano_rgb (canvas w*h*3) and pano_mask (w*h, 0/1) in host memory; either
 * may be NULL to skip that copy.  report may be NULL.  Synchronous, like the
 * reference. */
int stitch_b200_process(stitch_b200_ctx* ctx, const uint8_t* const* frames,
                        uint8_t* pano_rgb, uint8_t* pano_mask,
                        stitch_b200_report* report);

/* Pipelined variant of stitch_b200_process: enqueue one frame (upload of the
 * host frames on the context's copy stream, the frame on the compute stream,
 * download of the panorama into pano_rgb / pano_mask on a second copy
 * stream) and return a ticket without waiting.  Four frames can be in
 * flight (the context's pipeline slots): uploads and downloads of some
 * frames overlap the kernels of others.  Frames are processed in submission
 * order (the temporal state is sequential).  Host buffers must stay valid
 * until the ticket is waited.  Pinned buffers (stitch_b200_host_alloc or
 * stitch_b200_host_register) are copied by DMA directly; pageable ones (the
 * reference's std::vector frames) go through the slot's pinned staging ring,
 * filled and drained by the context's host copy workers, so the pipeline
 * keeps its frames in flight either way.  stitch_b200_wait blocks until the
 * ticket's panorama is in the caller's buffers and fills its report; a
 * ticket older than the last 8 retired frames is reported as MissingState.
 * Ticket numbers increase monotonically for the context's lifetime, across
 * update_geometry / update_maps / rerefine. */
int stitch_b200_submit(stitch_b200_ctx* ctx, const uint8_t* const* frames,
                       uint8_t* pano_rgb, uint8_t* pano_mask, long long* ticket);
int stitch_b200_wait(stitch_b200_ctx* ctx, long long ticket,
                     stitch_b200_report* report);

/* Masked input frames (Frame::mask, frame.hpp:44-47, e.g. PNG alpha,
 * image_io.cpp:120-127): masks[v] is NULL (view unmasked) or width*height
 * bytes, 0 = invalid pixel.  The warp skips masked taps exactly like
 * sample_bilinear (frame.cpp:95-104), and the canvas evaluates the
 * compose fold for every pixel of such a frame; results equal the
 * reference's process_frame on the same masked frames.  A masked view
 * without one valid warped pixel fails the frame with
 * STITCH_B200_EmptyProjection before it is enqueued, with the temporal state
 * untouched (warp_frame, geometry.cpp:79, throws before process_frame
 * changes any state, pipeline.cpp:270-277); submit then issues no ticket.
 * masks == NULL is stitch_b200_process / stitch_b200_submit. */
int stitch_b200_process_masked(stitch_b200_ctx* ctx, const uint8_t* const* frames,
                               const uint8_t* const* masks, uint8_t* pano_rgb,
                               uint8_t* pano_mask, stitch_b200_report* report);
int stitch_b200_submit_masked(stitch_b200_ctx* ctx, const uint8_t* const* frames,
                              const uint8_t* const* masks, uint8_t* pano_rgb,
                              uint8_t* pano_mask, long long* ticket);

/* Device-resident variant: frames[v] are device pointers; outputs stay in
 * the context (see stitch_b200_device_pano).  Ordered on the context's API
 * stream (stitch_b200_stream): inputs written there before the call are
 * seen, work enqueued there after it sees the outputs.  Returns without
 * synchronising unless report != NULL. */
int stitch_b200_process_device(stitch_b200_ctx* ctx,
                               const uint8_t* const* dev_frames,
                               stitch_b200_report* report);

/* Pipelined device-resident frames.  A context runs its pipeline slots
 * (stitch_b200_slots, 4 by default) on
 * their own streams; consecutive frames overlap except at the points where
 * the reference's temporal state orders them (the 3D-M window update, the
 * threshold history), which the slots chain in frame order.
 * process_device_async enqueues a frame without ordering against the API
 * stream; stitch_b200_fork makes subsequently enqueued frames wait for the
 * API stream's work so far, stitch_b200_join makes the API stream wait for
 * every frame enqueued so far.  The outputs of frame t stay valid until
 * frame t + slots is enqueued. */
int stitch_b200_process_device_async(stitch_b200_ctx* ctx, const uint8_t* const* dev_frames);
int stitch_b200_fork(stitch_b200_ctx* ctx);
int stitch_b200_join(stitch_b200_ctx* ctx);

/* Device pointers of the context's last panorama (rgb w*h*3, mask w*h). */
int stitch_b200_device_pano(const stitch_b200_ctx* ctx, uint8_t** rgb,
                            uint8_t** mask);

/* The CUDA stream (cudaStream_t) the context enqueues on. */
void* stitch_b200_stream(const stitch_b200_ctx* ctx);
int stitch_b200_synchronize(stitch_b200_ctx* ctx);

/* Number of kernel launches one processed frame issues. */
int stitch_b200_launches_per_frame(const stitch_b200_ctx* ctx);

/* Profiling: run one frame's launch plan eagerly (not as a graph) on the
 * context stream with a CUDA event pair around every kernel launch.
 * dev_frames as for stitch_b200_process_device.  Writes up to max_ops
 * (kernel-kind, milliseconds) pairs and returns the number of launches, or
 * a negative status.  Kinds: 0 expand_rgba, 1 crop_warp, 2 pair_color
 * (stats + solve), 4 flow_prepare, 5 pyr_down, 6 hs_linearize, 7 hs_sweeps,
 * 8 canvas_balance, 10 tone.  Advances the temporal state like a processed frame. */
int stitch_b200_profile_frame(stitch_b200_ctx* ctx,
                              const uint8_t* const* dev_frames, int max_ops,
                              int* kinds, float* ms);

/* ---- frame ingress / egress ----
 * PPM (P6, maxval 255) I/O, replacing read_ppm / write_ppm
 * (proj/src/image_io.cpp:61-85, header tokens with '#' comments as
 * read_ppm_token :19-37); failures return IoError like the reference's
 * StitchError(IoError).  read_ppm writes the raster into rgb (capacity
 * bytes, e.g. a pinned buffer) and the size into width/height; rgb == NULL
 * reads the header only.  PNG needs libpng, which this build does not have. */
int stitch_b200_ppm_info(const char* path, int* width, int* height);
int stitch_b200_read_ppm(const char* path, uint8_t* rgb, size_t capacity, int* width,
                         int* height);
int stitch_b200_write_ppm(const char* path, int width, int height, const uint8_t* rgb);
/* PNG, replacing read_png / write_png (image_io.cpp:87-165), on zlib (libpng
 * is not in this image).  Read: palette / grey / 16-bit expanded to 8-bit RGB
 * as libpng's expand + strip_16 + gray_to_rgb; alpha 0 (or tRNS) marks the
 * pixel invalid.  rgb (capacity bytes) and mask (mask_capacity bytes, 0/1,
 * all 1 without transparency) may be NULL to query the size; has_mask = 1
 * when some pixel is transparent.  Interlaced files are an IoError.  Write:
 * 8-bit RGB, or RGBA with alpha 255 / 0 from mask when mask != NULL. */
int stitch_b200_read_png(const char* path, uint8_t* rgb, size_t capacity, uint8_t* mask,
                         size_t mask_capacity, int* width, int* height, int* has_mask);
int stitch_b200_write_png(const char* path, int width, int height, const uint8_t* rgb,
                          const uint8_t* mask);
/* sequence_name (image_io.cpp:194-199): stem + "_%06d" + ext into out. */
int stitch_b200_sequence_name(const char* stem, int index, const char* ext, char* out,
                              size_t capacity);

typedef struct {
  long long frames;     /* panoramas written */
  double seconds;       /* wall time of the whole run */
  double read_seconds;  /* summed per-file read time (reader threads) */
  double write_seconds; /* summed per-file write time (writer threads) */
} stitch_b200_files_stats;

/* run_sequence (pipeline.hpp:90-92, pipeline.cpp:364-412) with file sources
 * and sink: view_dirs[v] holds view v's numbered image sequence
 * (list_sequence, image_io.cpp:181-192: the .ppm / .png files sorted by name;
 * a PNG with transparent pixels is a masked frame and runs with its mask,
 * stitch_b200_submit_masked);
 * frame t of every view is stitched in order and the panorama written to
 * out_dir/<stem>_%06d<ext> (ext ".ppm" (NULL) or ".png" with the mask as
 * alpha; out_dir NULL: not written).  One reader thread per
 * view reads straight into pinned staging, frames run four in flight through
 * stitch_b200_submit / stitch_b200_wait, four writer threads encode the
 * panoramas.  max_frames <= 0: every frame present in all views.  reports
 * (optional) receives one FrameReport per frame. */
int stitch_b200_run_files(stitch_b200_ctx* ctx, const char* const* view_dirs,
                          const char* out_dir, const char* stem, const char* ext, int max_frames,
                          stitch_b200_report* reports, stitch_b200_files_stats* stats);

/* Number of views / a view's camera size of a context. */
int stitch_b200_n_views(const stitch_b200_ctx* ctx);
/* Pipeline slots (frames that can be in flight) of the context: 4 unless
 * STITCH_B200_SLOTS (2..8) was set when it was built. */
int stitch_b200_slots(const stitch_b200_ctx* ctx);
int stitch_b200_view_size(const stitch_b200_ctx* ctx, int view, int* width, int* height);
/* Validates one frame set before process/submit: n must equal the configured
 * views and every frame must have the size its view was initialized with
 * (InputMismatch otherwise).  masks (may be NULL) are accepted: frames that
 * carry masks go through stitch_b200_process_masked / submit_masked.  The
 * C++ and Python mirrors call it on every frame set. */
int stitch_b200_check_frames(const stitch_b200_ctx* ctx, int n, const int* widths,
                             const int* heights, const uint8_t* const* masks);
/* Set the calling thread's last error; returns code. */
int stitch_b200_set_error(int code, const char* what);

/* Pinned host memory helpers (cudaHostAlloc / cudaFreeHost). */
void* stitch_b200_host_alloc(size_t bytes);
void stitch_b200_host_free(void* p);
/* Page-lock a caller-owned buffer the caller keeps for the context's
 * lifetime (its frame / output buffers), so submit/process copy it by DMA
 * instead of through the context's pinned staging ring; unregister before
 * freeing it. */
int stitch_b200_host_register(void* p, size_t bytes);
/* Test entry (host only): `rounds` back-to-back batches through the host
 * copy pool that stages pageable buffers, every byte verified. */
int stitch_b200_debug_copy_pool(int workers, int rounds, size_t bytes);
int stitch_b200_host_unregister(void* p);
/* Device memory helpers for callers without another allocator. */
void* stitch_b200_device_alloc(int device, size_t bytes);
void stitch_b200_device_free(void* p);
int stitch_b200_memcpy_h2d(void* dst, const void* src, size_t bytes);
int stitch_b200_memcpy_d2h(void* dst, const void* src, size_t bytes);

/* ---- per-stage debug readback of the last processed frame ---- */
/* Raw warped crops of pair k (side 0 = view, 1 = partner), bounds-sized,
 * RGB8 + mask, before color correction. */
int stitch_b200_debug_crop(stitch_b200_ctx* ctx, int k, int side,
                           int corrected, uint8_t* rgb, uint8_t* mask);
/* Final level-0 flow of pair k, dir 0 = view->partner, 1 = partner->view,
 * zeroed at invalid pixels (flow.cpp:178-185). */
int stitch_b200_debug_flow(stitch_b200_ctx* ctx, int k, int dir, float* u,
                           float* v);
/* Pre-balance panorama (after composition). */
int stitch_b200_debug_prebalance(stitch_b200_ctx* ctx, uint8_t* rgb,
                                 uint8_t* mask);
/* Full warped view v over the canvas (evaluated on demand with the same
 * device sampler, raw, before color correction). */
int stitch_b200_debug_warp_view(stitch_b200_ctx* ctx, int view,
                                const uint8_t* host_frame, uint8_t* rgb,
                                uint8_t* mask);

/* The synthetic scene generator (the reference's SynthScene, test and bench
 * inputs) is not part of this library: include/stitch_synth.h,
 * libstitch_synth.so. */

#ifdef __cplusplus
}
#endif
#endif
