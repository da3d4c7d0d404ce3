// kernels.cuh -- descriptor tables shared by the host context and the
// sm_100a kernels of the per-frame stitching path.
//
// HBM layout of one context (one panorama stream):
//   frames[v]      RGB8 interleaved, W*H*3 bytes (inputs; reused every frame)
//   crop_raw[k][s] uchar4 (r,g,b,valid) over pair k's bounds, s=0 view, 1 partner
//   crop_cor[k][s] same after the per-view 3x3 colour matrix
//   pyr[k][s][l]   float luma pyramid of crop_cor
//   flow[k][d]     float u/v ping-pong planes (level-0 sized, reused per level)
//   pano           uchar4 per canvas pixel (pre-balance), flat row-major
//   out_rgb/mask   balanced panorama in the reference's Frame layout
#pragma once

#include <cuda_runtime.h>

#include <mutex>

#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <utility>
#include <vector>

#include "stitch_b200.h"

namespace stitch_b200_dev {

constexpr int kMaxViews = STITCH_B200_MAX_VIEWS;
constexpr int kMaxPairs = STITCH_B200_MAX_PAIRS;
constexpr int kMaxLevels = 16;
constexpr int kMaxTasks = 2 * kMaxPairs;

struct ViewDesc {
  int width, height;
  int bbox[4];  // x0,y0,x1,y1 of the view's valid canvas footprint
  int gap[2];   // empty columns [gap0, gap1) inside bbox (wrapped ring views)
  double inv[9];
};

struct PairDesc {
  int view, partner;
  int x0, y0, w, h;  // bounds
  int flow_ok;       // 0: crop below 16x16 -> zero flow (pipeline.cpp:317-320)
  const float* theta_i;
  uchar4* crop_raw[2];
  uchar4* crop_cor[2];
  float* pyr[2][kMaxLevels];
  int levels;                // pyramid levels of the pair's flow (0: no flow)
  const float2* flow_uv[2];  // final level-0 flow (u, v), dir 0: view->partner
};

// Per-pair integer moments of one frame (k_pair_stats -> k_pair_solve).
struct PairStats {
  unsigned int hs[3][256];   // source (view) histogram
  unsigned int hr[3][256];   // reference (partner) histogram
  unsigned long long s[6][256];  // S_{a|b}[v] = sum_{x_b = v} x_a, (a,b) a!=b
  unsigned long long n;
};

// 3D-M window entry: exact integer moments of one frame
// (TransferWindow::Entry, color_transfer.hpp:43-46, reduced to X^T X, X^T Y).
struct WindowEntry {
  unsigned long long xtx[9];
  unsigned long long xty[9];
  unsigned long long n;
};

struct PairWindow {
  WindowEntry e[3];  // newest first
  int size;
  int capacity;
};

struct DevReport {
  long long frame_index;
  double m[kMaxPairs][9];
  int rank_deficient[kMaxPairs];
  int m1[3], m2[3];
  int balanced;
};

struct BalanceState {
  int n;  // history entries (<= 3), newest last
  int m1[3][3], m2[3][3];
};

// The per-frame part of the geometry, rewritten for every frame: the device
// RGB8 inputs, their masks (Frame::mask, frame.hpp:44-47: W*H bytes, 0 =
// invalid; nullptr = unmasked view) and whether this frame carries any mask.
// A masked frame's samplers skip masked taps (frame.cpp:95-104) and the
// canvas evaluates every pixel's fold instead of the geometry-only class map.
struct FrameTable {
  const std::uint8_t* frames[kMaxViews];
  const std::uint8_t* masks[kMaxViews];
  int masked;
};

struct Geometry {
  FrameTable in;                          // per frame
  uchar4* rgba[kMaxViews];                // the inputs expanded to RGBA8 (.w = valid)
  // canvas lift (extension): 0 planar (x+offx, y+offy, 1); 1 cylindrical
  // (sin t[x], h[y], cos t[x]) from host-computed tables
  int projection;
  const double* lift_sin;
  const double* lift_cos;
  const double* lift_h;
  int canvas_w, canvas_h;
  double offx, offy;
  int n_views, reference, n_pairs;
  int weighting;  // 0 own, 1 cross
  ViewDesc views[kMaxViews];
  PairDesc pairs[kMaxPairs];
  int pair_depth[kMaxPairs];
  // balance config
  double lambda, gamma_dark, gamma_bright;
  int target_black, target_white;
  int curve_ok;
};

// Linearisation of one warp iteration (refine_level, flow.cpp:84-108) for
// one (pair, direction) task at one level: u0 (zero / previous flow /
// coarser flow upsampled, flow.cpp:163-167) -> warped image bw -> the
// per-pixel Jacobi constants gx, gy, c = it - gx*u0 - gy*v0 and
// denom = alpha2 + gx*gx + gy*gy, written as planes.
struct PrepTask {
  const float* a;  // luma of the first image at this level
  const float* b;  // luma of the second image
  int mode;        // 0: u0 = 0, 1: u0 = uv_in, 2: upsample uv_in from wc x hc
  const float2* uv_in;
  int wc, hc;
  int w, h;
  float2* uv0_out;  // modes 0 and 2: u0 materialised here (the sweeps' start state)
  float4* kq;  // Jacobi constants per pixel: (gx, gy, c, denom)
};

// One segment of Jacobi sweeps (flow.cpp:109-134) on constant planes.
// Compact, launch-constant descriptors of the canvas and crop-warp passes,
// passed by value (__grid_constant__ kernel parameter, read through the
// constant bank with warp-uniform indices).
struct CanvasView {
  double inv[9];
  const uchar4* rgba;
  int w, h;
  int bbox[4];
  int gap[2];
  int f32;  // experiment (STITCH_B200_WARP_F32): FP32 interior weights and sums
};

struct CanvasPair {
  int view, partner, x0, y0, w, h;
  const float* theta;
  uchar4* crop_raw[2];
  const uchar4* crop_cor[2];
  const float2* fuv[2];
};

struct CanvasParams {
  const int* masked;  // -> the slot's FrameTable::masked (device, per frame)
  int cw, ch, ref, np, weighting;
  double offx, offy;
  int projection;
  const double* lift_sin;
  const double* lift_cos;
  const double* lift_h;
  CanvasView views[kMaxViews];
  CanvasPair pairs[kMaxPairs];
  // per canvas pixel, from the geometry alone (k_canvas_class): the view the
  // compose fold takes the pixel from when it lies outside every pair's
  // bounds, kClassFold inside some pair's bounds, kClassNone if no view
  // covers it; nullptr = evaluate the fold everywhere
  const std::uint8_t* cls;
};
constexpr std::uint8_t kClassFold = 254, kClassNone = 255;

struct HsTask {
  float4* kq;  // Jacobi constants (gx, gy, c, denom) per pixel: read by plain
               // segments, written (output tile) by a segment that fuses the
               // linearisation
  const float2* uv_in;  // state (u, v) at the start of the segment (fused:
                        // the u0 source of lin_mode, see PrepTask::mode)
  float2* uv_out;
  int w, h;
  // fused linearisation (first segment of a warp iteration)
  const float* lin_a;  // luma of the first / second image at this level
  const float* lin_b;
  int lin_mode;  // 0: u0 = 0, 1: u0 = uv_in, 2: uv_in upsampled from wc x hc
  int wc, hc;
  // epilogue linearisation (last segment of a warp iteration): the next warp
  // iteration's constants, from lin_a / lin_b and this segment's result
  float4* kq_next;
  // TMA tensor map (CUtensorMap, 64-byte aligned, in device memory) of the
  // kq plane as a 4w x h float tensor, for the TMA-staged plain segment
  const void* kq_map;
};

struct PyrTask {
  const float* src;
  int sw, sh;
  float* dst;
  int w, h;
};

// mutable per-context device state
// Temporal state of one stream (PipelineState's windows, threshold history
// and frame counter): shared by the pipeline slots, updated in frame order.
struct TemporalState {
  PairWindow windows[kMaxPairs];
  BalanceState balance;
  long long frame_counter;
};

// Per-slot frame state: scratch accumulators, this frame's colour matrices,
// LUT and report, plus pointers into the shared TemporalState.
struct DevState {
  PairStats stats[kMaxPairs];
  PairWindow* windows;          // -> TemporalState::windows
  double mview[kMaxViews][9];  // colour matrix applied to each view
  unsigned int pano_hist[3][256];
  BalanceState* balance;        // -> TemporalState::balance
  unsigned char lut[3][256];
  DevReport report;
  long long* frame_counter;     // -> TemporalState::frame_counter
  unsigned int pair_done[kMaxPairs];  // CTA completion counters (last-CTA solve)
  unsigned int canvas_done;
};

// integer experiment / tuning switch from the environment (read once by the
// callers, which keep it in a static)
inline int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

// ---- launchers (kernels.cu) ----
void launch_expand(const Geometry* g, int n_views, long long max_px, cudaStream_t s);
void launch_crop_warp(const CanvasParams& P, int max_w, int max_h, cudaStream_t s);
int launch_pair_color(const Geometry* g, DevState* st, const int* pair_list, int n,
                       int max_crop_px, cudaStream_t s);
void launch_flow_prepare(const Geometry* g, DevState* st, int n_pairs, int max_crop_px,
                         cudaStream_t s);
void launch_pyr_down(const PyrTask* tasks, int n, int max_px, cudaStream_t s);
// flow_prepare + the first kPyrFused pyramid levels in one launch
constexpr int kPyrFused = 4;
void launch_flow_prepare_pyr(const Geometry* g, DevState* st, int n_pairs, int max_w, int max_h,
                             cudaStream_t s);
int pyr_fuse_wanted();
size_t hs_smem_bytes(int sweeps);
// how many launches (sweep segments) one warp iteration of `sweeps` uses
int hs_segments(int sweeps);
// segment lengths of one warp iteration at a level (tasks n, max w x h)
std::vector<int> hs_split(int n, int max_w, int max_h, int sweeps);
cudaError_t prepare_hs(int sweeps);
// TMA-staged plain segments (STITCH_B200_HS_TMA): whether they are on, and
// the CUtensorMap (128 bytes) of a w x h float4 plane
bool hs_tma_wanted();
bool encode_kq_map(void* map128, const float4* kq, int w, int h);
void launch_hs_prepare(const PrepTask* tasks, int n, int max_w, int max_h, float alpha2,
                       cudaStream_t s);
// fuse_lin: 0 plain segment; 1 the segment first linearises the warp
// iteration (HsTask lin_* fields); 2 the segment also linearises the next
// warp iteration on its output tile (HsTask lin_a, lin_b, kq_next)
void launch_hs_iter(const HsTask* tasks, int n, int max_w, int max_h, int sweeps, int fuse_lin,
                    float alpha2, cudaStream_t s);
// the fused linearisation serves segments of up to this many sweeps
int hs_fuse_max_sweeps();
// whether the first segment of a warp iteration with these dimensions should
// fuse the linearisation (the launch it would use supports and profits from it)
int hs_fuse_wanted(int n, int max_w, int max_h, int sweeps);
// whether a warp iteration's last segment (`sweeps` long) should linearise
// the next warp iteration in its epilogue
int hs_elin_wanted(int n, int max_w, int max_h, int sweeps);
// mode 0: whole canvas; 1: outside every pair's bounds (flow-independent);
// 2: inside the bounds.  Modes 1 + 2 together cover the canvas once.
int launch_canvas(const CanvasParams& P, const Geometry* g, DevState* st, uchar4* pano,
                  int num_sms, cudaStream_t s);
void launch_tone(const DevState* st, const uchar4* pano, long long n_px,
                 std::uint8_t* out_rgb, std::uint8_t* out_mask, cudaStream_t s);
void launch_warp_view(const Geometry* g, int view, const uchar4* frame, std::uint8_t* rgb,
                      std::uint8_t* mask, cudaStream_t s, bool masked = false);
void launch_expand_one(const std::uint8_t* rgb, uchar4* rgba, long long n_px, cudaStream_t s,
                       const std::uint8_t* mask = nullptr);
void launch_warp_mask(const Geometry* g, int view, std::uint8_t* mask, cudaStream_t s);
// Coverage of masked frames (warp_frame's EmptyProjection, geometry.cpp:79):
// for each listed view, does its masked frame give at least one valid warped
// pixel inside rect?  Sets bit view of *covered (zeroed by the caller).
struct MaskSet {
  int n;
  int view[kMaxViews];
  const std::uint8_t* mask[kMaxViews];  // W x H bytes, nonzero = valid
  int rect[kMaxViews][4];               // canvas x0, y0, x1, y1 to scan
};
void launch_mask_coverage(const Geometry* g, int projection, const MaskSet& ms, long long max_px,
                          unsigned* covered, cudaStream_t s);
// the canvas class map of CanvasParams::cls (init time, geometry only)
void launch_canvas_class(const CanvasParams& P, std::uint8_t* cls, cudaStream_t s);
// test entry: n tone curves (build_curve) for the given (m1[i], m2[i])
void launch_debug_tone_curves(int n, const int* m1, const int* m2, double gamma_dark,
                              double gamma_bright, double tb, double tw, std::uint8_t* out,
                              cudaStream_t s);

// ---- feature refinement image work (features_kernels.cu) ----
struct FeatPoint {
  double x, y, scale, response;  // Keypoint (features.hpp)
};
// One warped view: the integral image of its quantized gray, then
// detect + describe over a search region (keypoints in the reference's
// order, 64 floats per descriptor).
class FeatView {
 public:
  FeatView();
  ~FeatView();
  FeatView(const FeatView&) = delete;
  FeatView& operator=(const FeatView&) = delete;
  cudaError_t build(const std::uint8_t* d_rgb, int w, int h, cudaStream_t s);
  cudaError_t detect_describe(int rx0, int ry0, int rx1, int ry1, double threshold,
                              std::vector<FeatPoint>& kps, std::vector<float>& desc,
                              cudaStream_t s) const;

 private:
  struct Impl;
  Impl* impl;
};
// match (features.cpp:181-234) on the device: per a the ratio-tested
// nearest b (-1 when rejected) and its distance, per b the nearest a.
cudaError_t feat_match(const std::vector<float>& da, const std::vector<float>& db, int na, int nb,
                       double ratio, std::vector<int>& best_b, std::vector<double>& best_dist,
                       std::vector<int>& best_a, cudaStream_t s);

// ---- quality metrics (metrics_kernels.cu) ----
// Quality-metric scratch: grow-only device buffers and a stream per device,
// reused across calls (no allocation or free per metric call); callers hold
// mu for the duration of a metric.
struct MetricsWorkspace {
  enum { kPackRgb, kPackMask, kPackA, kPackB, kPsnrAcc, kSsimTmp, kSsimTerm, kSsimCnt, kSsimValid,
         kSsimSum, kSlots };
  std::mutex mu;
  cudaStream_t s = nullptr;
  void* p[kSlots] = {};
  size_t cap[kSlots] = {};
  cudaError_t get(int slot, size_t bytes, void** out);
};
MetricsWorkspace& metrics_workspace();  // the current device's

cudaError_t gpu_psnr_parts(MetricsWorkspace& ws, const uchar4* a, const uchar4* b, int n,
                           unsigned long long* sse, unsigned long long* count, cudaStream_t s);
cudaError_t gpu_ssim_parts(MetricsWorkspace& ws, const uchar4* a, const uchar4* b, int w, int h,
                           double* sum, long long* count, cudaStream_t s);
// which: 0 / 1 = the workspace's first / second packed frame
cudaError_t gpu_pack_rgba(MetricsWorkspace& ws, int which, const std::uint8_t* rgb_host,
                          const std::uint8_t* mask_host, int n, uchar4** out, cudaStream_t s);

// ---- init-time geometry on the device (geometry_kernels.cu) ----
struct ViewFootprint {
  int bbox[4] = {0, 0, 0, 0};  // bbox of the warp mask
  int gap[2] = {0, 0};         // widest empty column run inside it
  bool empty = true;
  bool masked_empty = false;   // a masked first frame warps to no pixel
};
struct PairGeometry {
  bool ok = false;             // the pair's masks overlap
  int bounds[4] = {0, 0, 0, 0};
  std::vector<float> theta;    // blend weight theta_i over the bounds
};
// Warp masks of every view (launch_warp_mask), view footprints, and for each
// (view, partner) pair its overlap bounds and chamfer blend weights.
// first_rgba: the first frames expanded to RGBA with their masks as alpha
// (per view, nullptr = unmasked): the pairs' bounds and weights then follow
// those frames' masked warps, as rebuild_pair_geometry warps first_frames
// (pipeline.cpp:181-205); the view footprints stay the geometry's.
// lift_*: the cylindrical lift tables (projection 1), else unused.
cudaError_t gpu_init_geometry(const Geometry& geom, const double* lift_s, const double* lift_c,
                              const double* lift_h, int n_lift_x, int n_lift_y, int n_views,
                              const std::vector<std::pair<int, int>>& pairs,
                              std::vector<ViewFootprint>& views, std::vector<PairGeometry>& out,
                              const std::vector<const uchar4*>* first_rgba = nullptr);

}  // namespace stitch_b200_dev
