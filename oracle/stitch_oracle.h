/*
 * stitch_oracle.h -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference's per-frame stitching path
 * (/root/reference/proj/src/{frame,histogram,geometry,color_transfer,
 * color_balance,flow,pipeline}.cpp) plus the init-time geometry it needs.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load this library, and only as the checker or
 * as the timed CPU baseline.  The B200 product never links or calls it.
 *
 * Parity status: the reference itself cannot be built here (it needs
 * Eigen3, libpng and doctest, all absent), so this
 * restatement is pinned against the reference's shipped known-answer tests
 * (proj/tests/test_imaging.cpp:34-191) and the SPEC.md examples restated in
 * tests/test_oracle_pins.py.  Results at the Eigen boundary (3x3 products,
 * inverse, JacobiSVD, LDLT) follow Eigen's published algorithms with a
 * fixed left-to-right summation order: PARITY UNPINNED at the last ulp there.
 *
 * N-view extension (not in the reference, which caps views at 3): views > 3
 * use an adjacent-pair chain (partner = neighbour toward the reference,
 * pairs ordered outward); for <= 3 views the star topology of
 * pipeline.cpp:233-239 is used unchanged.
 */
#ifndef STITCH_ORACLE_H
#define STITCH_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SO_MAX_VIEWS 16

/* ErrorCode, types.hpp:9-27 (same order). */
enum so_error {
  SO_OK = -1,
  SO_EmptyRegion = 0,
  SO_EmptyHistogram,
  SO_RankDeficient,
  SO_RegionTooSmall,
  SO_InsufficientMatches,
  SO_NoConsensus,
  SO_ShapeMismatch,
  SO_NoOverlap,
  SO_SingularHomography,
  SO_DegeneratePose,
  SO_EmptyProjection,
  SO_MissingState,
  SO_TooSmall,
  SO_ConfigError,
  SO_ConfigurationError,
  SO_InputMismatch,
  SO_IoError
};

/* Frame, frame.hpp:17-57: RGB8 interleaved, optional 0/1 mask (NULL = all
 * pixels valid). */
typedef struct {
  int width, height;
  uint8_t* data;
  uint8_t* mask;
} so_frame;

/* Region, types.hpp:47-62: half-open [x0,x1) x [y0,y1). */
typedef struct {
  int x0, y0, x1, y1;
} so_region;

typedef struct {
  uint32_t bins[3][256];
  uint64_t total;
} so_hist;

typedef struct {
  double fx, fy, cx, cy;
  double rotation[9]; /* row-major world->camera */
  double translation[3];
} so_camera;

typedef struct {
  int n_views;
  int reference;
  int width[SO_MAX_VIEWS], height[SO_MAX_VIEWS];
  so_camera cams[SO_MAX_VIEWS];
  /* BalanceConfig, color_balance.hpp:19-25 */
  double lambda, gamma_dark, gamma_bright;
  int target_black, target_white;
  /* FlowOptions, flow.hpp:29-34 */
  int flow_levels, flow_iterations;
  double smoothness;
  int window_capacity;
  int fuse_weighting; /* 0 = own (OwnWeightOnOwnFlow), 1 = cross */
  int topology;       /* 0 = auto (star <= 3 views, chain otherwise), 1 = star, 2 = chain,
                         3 = ring chain */
  int threads;
  int keep_debug;     /* keep raw warped views + flows of the last frame */
  /* extension: 0 planar (the reference), 1 cylindrical 360-degree canvas
   * (cameras share a centre; A_v = K_v R_v R_ref^T applied to
   * (sin t, h, cos t); samples behind the camera are invalid) */
  int projection;
  double cyl_focal;   /* pixels per radian; 0 = reference fx */
  /* RefineOptions (pipeline.hpp:23-31) + StitchConfig.seed; refinement runs
   * in so_initialize_frames only (it needs the first frames) */
  int refine_enabled;
  double refine_margin;
  int ransac_iters;
  double inlier_px;
  double detect_threshold;
  double match_ratio;
  unsigned long long seed;
} so_config;

typedef struct {
  long frame_index;
  int n_pairs;
  double m[SO_MAX_VIEWS][9]; /* row-major M per pair */
  int rank_deficient[SO_MAX_VIEWS];
  int threshold_m1[3], threshold_m2[3];
  int balanced; /* 0 when the panorama histogram was empty */
  double stage_seconds[4];
} so_report;

typedef struct so_state so_state;

/* ---- imaging primitives ---- */
uint8_t so_quantize_channel(double v);
int so_sample_bilinear(const so_frame* f, double x, double y, float rgb[3]);
int so_compute_histogram(const so_frame* f, so_region r, so_hist* out);
int so_cdf(const so_hist* h, double out[3][256]);
void so_inverse3(const double m[9], double out[9]);
double so_det3(const double m[9]);

/* ---- geometry ---- */
int so_warp_frame(const so_frame* src, const double inv[9], int cw, int ch,
                  double offx, double offy, int threads, so_frame* out);
/* generalised warp: lift = NULL -> planar (x+offx, y+offy, 1); else the
 * cylindrical lift tables lsin[cw], lcos[cw], lh[ch] */
int so_warp_frame_lift(const so_frame* src, const double a[9], int cw, int ch,
                       double offx, double offy, const double* lsin,
                       const double* lcos, const double* lh, int threads,
                       so_frame* out);

/* ---- color transfer ---- */
int so_histogram_specification(const so_hist* src, const so_hist* ref,
                               uint8_t lut[3][256]);
/* rows: n x 3 doubles each, one window entry per (src,tgt) pair, newest
 * first.  Returns SO_OK or SO_RankDeficient / SO_MissingState. */
int so_solve_color_matrix(int entries, const int* rows,
                          const double* const* src, const double* const* tgt,
                          double m[9], double* min_singular);
void so_sym3_eigen(const double a[9], double ev[3]);
void so_ldlt_solve3(const double a[9], const double b[9], double x[9]);
void so_apply_color_matrix_rows(so_frame* f, const double m[9], int threads);

/* ---- color balance ---- */
int so_find_thresholds(const so_hist* h, double lambda, int m1[3], int m2[3]);
void so_smooth_thresholds(int n, const int (*m1)[3], const int (*m2)[3],
                          int out_m1[3], int out_m2[3]);
double so_balance_curve_value(double x, int m1, int m2, double gamma_dark,
                              double gamma_bright, int tb, int tw);
int so_build_curve(const int m1[3], const int m2[3], double gamma_dark,
                   double gamma_bright, int tb, int tw, uint8_t lut[3][256]);

/* ---- flow ---- */
int so_dense_flow(const so_frame* a, const so_frame* b, int levels,
                  int iterations, double smoothness, int threads, float* u,
                  float* v);
void so_blend_weights(const so_frame* wi, const so_frame* wj, so_region b,
                      float* theta_i, float* theta_j);
int so_flow_fuse(const so_frame* ri, const so_frame* rj, const float* uij,
                 const float* vij, const float* uji, const float* vji,
                 const float* theta_i, const float* theta_j, int weighting,
                 so_frame* out);
int so_compose_panorama(const so_frame* wi, const so_frame* wj,
                        const so_frame* fused, so_region overlap,
                        so_frame* out);

/* ---- feature refinement (features.cpp, features_oracle.cpp) ---- */
typedef struct {
  double x, y, scale, response;
} so_keypoint;
typedef struct {
  int index_a, index_b;
  double distance, ax, ay, bx, by;
} so_match_pair;
typedef struct {
  double s_x, s_y, t_x, t_y;
} so_similarity;
/* *out is malloc'ed (free()); SO_RegionTooSmall below 32x32 */
int so_detect(const so_frame* f, so_region r, double threshold, so_keypoint** out, int* n_out);
void so_describe(const so_frame* f, const so_keypoint* kps, int n, float* desc /* n*64 */);
/* out: capacity na; returns the match count */
int so_match(const float* da, int na, const float* db, int nb, const so_keypoint* ka,
             const so_keypoint* kb, double ratio, so_match_pair* out);
int so_ransac(const so_match_pair* m, int n, int iterations, double inlier_px, double min_scale,
              double max_scale, unsigned long long seed, so_similarity* out);

/* ---- pipeline (pipeline.cpp:209-360) ---- */
so_state* so_initialize(const so_config* cfg, int* err);
/* initialize() with the first frames: feature refinement when
 * cfg->refine_enabled (pipeline.cpp:241-255, refine_pair :114-179) */
so_state* so_initialize_frames(const so_config* cfg, const so_frame* first_frames, int* err);
/* the (possibly refined) view->reference maps and whether pair k's
 * refinement was kept (0) or fell back to the unrefined map (1) */
int so_state_refine_warning(const so_state* s, int k);
void so_destroy(so_state* s);
int so_process_frame(so_state* s, const so_frame* frames, so_frame* pano,
                     so_report* rep);

/* state inspection (for parity of the init-time geometry) */
void so_state_canvas(const so_state* s, int* w, int* h, double* offx,
                     double* offy);
void so_state_map(const so_state* s, int view, double h[9], double inv[9]);
int so_state_n_pairs(const so_state* s);
void so_state_pair(const so_state* s, int k, int* view, int* partner,
                   so_region* bounds);
void so_state_pair_weights(const so_state* s, int k, float* theta_i);
void so_state_view_bbox(const so_state* s, int view, so_region* bbox);
/* intermediates of the last processed frame (for per-stage parity) */
int so_state_last_flow(const so_state* s, int k, int dir, float* u, float* v);
int so_state_last_warped(const so_state* s, int view, uint8_t* rgb,
                         uint8_t* mask);

/* ---- quality metrics (metrics.cpp:9-155) ---- */
/* PSNR in dB over jointly valid pixels, channels pooled; +inf for identical
 * inputs.  Returns SO_OK, SO_ShapeMismatch or SO_EmptyRegion. */
int so_psnr(const so_frame* a, const so_frame* b, double* out);
/* mean SSIM on Rec.601 luma, 11x11 Gaussian (sigma 1.5), windows with fully
 * jointly valid support.  SO_ShapeMismatch, SO_TooSmall or SO_EmptyRegion. */
int so_ssim(const so_frame* a, const so_frame* b, double* out);

/* helpers */
void so_free_frame(so_frame* f);

#ifdef __cplusplus
}
#endif
#endif
