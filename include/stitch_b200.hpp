// stitch_b200.hpp -- C++ mirror of the reference pipeline API over the C ABI.
//
// Same names, argument meaning and error behaviour as
//   /root/reference/proj/include/stitch/pipeline.hpp:17-92   (StitchConfig,
//       PipelineState, initialize, process_frame, run_sequence)
//   /root/reference/proj/include/stitch/report.hpp:11-58     (Stage, FrameReport,
//       RunReport)
//   /root/reference/proj/include/stitch/types.hpp:9-62       (ErrorCode,
//       StitchError, Region)
//   /root/reference/proj/include/stitch/frame.hpp:17-57      (Frame)
// with Eigen types replaced by std::array so the header has no third-party
// dependency.  Header-only: everything crosses into libstitch_b200.so through
// the extern "C" entry points of stitch_b200.h, so the C++ ABI of the caller
// never has to match the library's.  Errors surface as StitchError, like the
// reference; stage failures inside a frame degrade (identity matrix, zero
// flow, unbalanced frame) and are reported, never thrown.
#pragma once

#include <array>
#include <chrono>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "stitch_b200.h"

namespace stitch_b200 {

// ---- types.hpp ----
enum class ErrorCode {
  EmptyRegion,
  EmptyHistogram,
  RankDeficient,
  RegionTooSmall,
  InsufficientMatches,
  NoConsensus,
  ShapeMismatch,
  NoOverlap,
  SingularHomography,
  DegeneratePose,
  EmptyProjection,
  MissingState,
  TooSmall,
  ConfigError,
  ConfigurationError,
  InputMismatch,
  IoError,
  // B200-side failures (no reference counterpart)
  DeviceError,
  Unsupported,
};

class StitchError : public std::runtime_error {
 public:
  StitchError(ErrorCode code, std::string message)
      : std::runtime_error(std::move(message)), code_(code) {}
  ErrorCode code() const noexcept { return code_; }

 private:
  ErrorCode code_;
};

inline void check(int status) {
  if (status == STITCH_B200_OK) return;
  ErrorCode code = ErrorCode::DeviceError;
  if (status >= 1 && status <= 17)
    code = static_cast<ErrorCode>(status - 1);
  else if (status == STITCH_B200_Unsupported)
    code = ErrorCode::Unsupported;
  throw StitchError(code, stitch_b200_last_error());
}

struct Region {
  int x0 = 0, y0 = 0, x1 = 0, y1 = 0;
  int width() const { return x1 - x0; }
  int height() const { return y1 - y0; }
  bool empty() const { return x1 <= x0 || y1 <= y0; }
};

// ---- frame.hpp ----
struct Frame {
  int width = 0;
  int height = 0;
  std::vector<std::uint8_t> data;  // width*height*3, R,G,B interleaved
  std::vector<std::uint8_t> mask;  // empty, or width*height 0/1

  Frame() = default;
  Frame(int w, int h, std::uint8_t fill = 0)
      : width(w), height(h), data(static_cast<std::size_t>(w) * h * 3, fill) {}
  bool has_mask() const { return !mask.empty(); }
  std::size_t pixel_count() const { return static_cast<std::size_t>(width) * height; }
};

// ---- geometry.hpp / color_balance.hpp / flow.hpp ----
struct CameraIntrinsics {
  double fx = 1.0, fy = 1.0, cx = 0.0, cy = 0.0;
};

struct CameraExtrinsics {
  std::array<double, 9> rotation{1, 0, 0, 0, 1, 0, 0, 0, 1};  // row-major world -> camera
  std::array<double, 3> translation{0, 0, 0};
};

struct BalanceConfig {
  double lambda = 0.05;
  double gamma_dark = 1.5;
  double gamma_bright = 1.5;
  int target_black = 0;
  int target_white = 255;
};

struct FlowOptions {
  int levels = 4;
  int iterations = 50;
  double smoothness = 15.0;
  int threads = 1;  // accepted for source compatibility; the GPU ignores it
};

enum class FuseWeighting { OwnWeightOnOwnFlow, CrossWeightOnOwnFlow };

// ---- pipeline.hpp ----
struct ViewSetup {
  std::string dir;
  CameraIntrinsics intrinsics;
  CameraExtrinsics extrinsics;
};

struct RefineOptions {
  // Feature refinement at initialize(): detection / description / matching on
  // the device, RANSAC on the host (stitch_b200_initialize_frames).  On by
  // default, like the reference (pipeline.hpp:24).
  bool enabled = true;
  double margin = 0.15;
  int ransac_iters = 500;
  double inlier_px = 2.0;
  double detect_threshold = 2e-4;
  double match_ratio = 0.8;
  int rerefine_every = 0;
};

struct StitchConfig {
  std::vector<ViewSetup> views;
  int reference = 0;
  BalanceConfig balance;
  FlowOptions flow;
  RefineOptions refine;
  int threads = 1;
  std::uint64_t seed = 0;
  int window_capacity = 3;
  FuseWeighting fuse_weighting = FuseWeighting::OwnWeightOnOwnFlow;
  std::string scene_id = "scene";
  int topology = 0;  // extension: 0 auto (star <= 3 views, chain beyond), 1 star, 2 chain
  int device = 0;
};

// ---- report.hpp ----
enum class Stage : int { GeometricWarping = 0, ColorCorrection = 1, LocalWarping = 2, ImageBlending = 3 };
constexpr int kStageCount = 4;

struct StageTimes {
  std::array<double, kStageCount> seconds{};
  double total() const {
    double t = 0.0;
    for (double s : seconds) t += s;
    return t;
  }
  double& operator[](Stage s) { return seconds[static_cast<int>(s)]; }
  double operator[](Stage s) const { return seconds[static_cast<int>(s)]; }
  StageTimes& operator+=(const StageTimes& o) {
    for (int i = 0; i < kStageCount; ++i) seconds[i] += o.seconds[i];
    return *this;
  }
};

using Matrix3d = std::array<double, 9>;  // row-major

struct FrameReport {
  long frame_index = 0;
  StageTimes times;
  std::vector<Matrix3d> color_matrices;
  std::vector<bool> rank_deficient;
  std::array<int, 3> threshold_m1{};
  std::array<int, 3> threshold_m2{};
};

struct RunReport {
  std::string scene_id;
  int threads = 1;
  long frames = 0;
  StageTimes totals;
  double wall_seconds = 0.0;
  std::vector<FrameReport> per_frame;
  std::string config_hash;
  bool refine_warning = false;
  double fps() const { return wall_seconds > 0 ? frames / wall_seconds : 0.0; }
};

// Device-resident pipeline state: owns one stitch_b200_ctx.
class PipelineState {
 public:
  PipelineState() = default;
  explicit PipelineState(stitch_b200_ctx* ctx, StitchConfig cfg)
      : ctx_(ctx, &stitch_b200_destroy), config(std::move(cfg)) {}
  stitch_b200_ctx* handle() const { return ctx_.get(); }
  int canvas_width() const {
    int w = 0;
    stitch_b200_canvas(ctx_.get(), &w, nullptr, nullptr, nullptr);
    return w;
  }
  int canvas_height() const {
    int h = 0;
    stitch_b200_canvas(ctx_.get(), nullptr, &h, nullptr, nullptr);
    return h;
  }
  int n_pairs() const { return stitch_b200_n_pairs(ctx_.get()); }
  // Re-refinement from new view->reference homographies (row-major, 9 per
  // view): canvas and pair geometry rebuilt on the device, temporal state
  // kept (run_sequence's rerefine branch, pipeline.cpp:395-406).
  void update_maps(const std::vector<std::array<double, 9>>& maps) {
    std::vector<double> flat;
    for (const auto& m : maps) flat.insert(flat.end(), m.begin(), m.end());
    check(stitch_b200_update_maps(ctx_.get(), flat.data()));
  }

 private:
  std::unique_ptr<stitch_b200_ctx, void (*)(stitch_b200_ctx*)> ctx_{nullptr, &stitch_b200_destroy};

 public:
  StitchConfig config;
  long frame_counter = 0;
};

struct ProcessResult {
  Frame panorama;
  FrameReport report;
};

inline stitch_b200_config to_c(const StitchConfig& config, const std::vector<Frame>& first) {
  stitch_b200_config c;
  stitch_b200_config_defaults(&c);
  c.n_views = static_cast<int>(config.views.size());
  c.reference = config.reference;
  for (std::size_t v = 0; v < config.views.size() && v < STITCH_B200_MAX_VIEWS; ++v) {
    c.width[v] = first[v].width;
    c.height[v] = first[v].height;
    const ViewSetup& s = config.views[v];
    c.cams[v].fx = s.intrinsics.fx;
    c.cams[v].fy = s.intrinsics.fy;
    c.cams[v].cx = s.intrinsics.cx;
    c.cams[v].cy = s.intrinsics.cy;
    for (int i = 0; i < 9; ++i) c.cams[v].rotation[i] = s.extrinsics.rotation[i];
    for (int i = 0; i < 3; ++i) c.cams[v].translation[i] = s.extrinsics.translation[i];
  }
  c.lambda = config.balance.lambda;
  c.gamma_dark = config.balance.gamma_dark;
  c.gamma_bright = config.balance.gamma_bright;
  c.target_black = config.balance.target_black;
  c.target_white = config.balance.target_white;
  c.flow_levels = config.flow.levels;
  c.flow_iterations = config.flow.iterations;
  c.smoothness = config.flow.smoothness;
  c.window_capacity = config.window_capacity;
  c.fuse_weighting = config.fuse_weighting == FuseWeighting::CrossWeightOnOwnFlow ? 1 : 0;
  c.topology = config.topology;
  c.refine_enabled = config.refine.enabled ? 1 : 0;
  c.refine_margin = config.refine.margin;
  c.ransac_iters = config.refine.ransac_iters;
  c.inlier_px = config.refine.inlier_px;
  c.detect_threshold = config.refine.detect_threshold;
  c.match_ratio = config.refine.match_ratio;
  c.seed = config.seed;
  return c;
}

// initialize (pipeline.hpp:73-74); with refine.enabled the first frames feed
// the feature refinement (pipeline.cpp:241-255).
inline PipelineState initialize(const StitchConfig& config, const std::vector<Frame>& first_frames) {
  const int n = static_cast<int>(config.views.size());
  if (n < 2 || n > STITCH_B200_MAX_VIEWS)
    throw StitchError(ErrorCode::ConfigurationError, "pipeline supports 2 to 16 views");
  if (first_frames.size() != config.views.size())
    throw StitchError(ErrorCode::ConfigurationError, "frame count does not match configured views");
  bool any_mask = false;
  for (const Frame& f : first_frames) {
    if (f.data.size() != f.pixel_count() * 3)
      throw StitchError(ErrorCode::InputMismatch, "frame data must be width*height*3 bytes");
    if (f.has_mask() && f.mask.size() != f.pixel_count())
      throw StitchError(ErrorCode::InputMismatch, "frame mask must be width*height bytes");
    any_mask = any_mask || f.has_mask();
  }
  stitch_b200_config c = to_c(config, first_frames);
  stitch_b200_ctx* ctx = nullptr;
  if (any_mask) {  // masked first frames decide the pair geometry (pipeline.cpp:181-205)
    std::vector<const std::uint8_t*> ptrs, masks;
    for (const Frame& f : first_frames) {
      ptrs.push_back(f.data.data());
      masks.push_back(f.has_mask() ? f.mask.data() : nullptr);
    }
    check(stitch_b200_initialize_frames_masked(&c, ptrs.data(), masks.data(), config.device, &ctx));
  } else if (config.refine.enabled) {
    std::vector<const std::uint8_t*> ptrs;
    for (const Frame& f : first_frames) ptrs.push_back(f.data.data());
    check(stitch_b200_initialize_frames(&c, ptrs.data(), config.device, &ctx));
  } else {
    check(stitch_b200_initialize(&c, config.device, &ctx));
  }
  return PipelineState(ctx, config);
}

// process_frame (pipeline.hpp:79-80): one frame through warp -> 3D-M colour
// -> flow -> blend -> balance on the GPU.
inline ProcessResult process_frame(PipelineState& state, const std::vector<Frame>& frames) {
  if (frames.size() != state.config.views.size())
    throw StitchError(ErrorCode::ConfigurationError, "frame count does not match configured views");
  std::vector<const std::uint8_t*> ptrs, masks;
  std::vector<int> ws, hs;
  for (const Frame& f : frames) {
    if (f.data.size() != f.pixel_count() * 3)
      throw StitchError(ErrorCode::InputMismatch, "frame data must be width*height*3 bytes");
    if (f.has_mask() && f.mask.size() != f.pixel_count())
      throw StitchError(ErrorCode::InputMismatch, "frame mask must be width*height bytes");
    ptrs.push_back(f.data.data());
    masks.push_back(f.has_mask() ? f.mask.data() : nullptr);
    ws.push_back(f.width);
    hs.push_back(f.height);
  }
  // sizes as initialized, no masked pixel (stitch_b200_check_frames)
  check(stitch_b200_check_frames(state.handle(), static_cast<int>(frames.size()), ws.data(),
                                 hs.data(), masks.data()));
  ProcessResult result;
  Frame& pano = result.panorama;
  pano.width = state.canvas_width();
  pano.height = state.canvas_height();
  pano.data.resize(pano.pixel_count() * 3);
  pano.mask.resize(pano.pixel_count());
  stitch_b200_report r;
  bool any_mask = false;
  for (const std::uint8_t* m : masks) any_mask = any_mask || m != nullptr;
  if (any_mask)  // Frame::mask: masked taps drop out (frame.cpp:95-104)
    check(stitch_b200_process_masked(state.handle(), ptrs.data(), masks.data(), pano.data.data(),
                                     pano.mask.data(), &r));
  else
    check(stitch_b200_process(state.handle(), ptrs.data(), pano.data.data(), pano.mask.data(), &r));
  FrameReport& rep = result.report;
  rep.frame_index = static_cast<long>(r.frame_index);
  for (int i = 0; i < kStageCount; ++i) rep.times.seconds[i] = r.stage_ms[i] * 1e-3;
  for (int k = 0; k < r.n_pairs; ++k) {
    Matrix3d m;
    for (int i = 0; i < 9; ++i) m[i] = r.color_matrices[k][i];
    rep.color_matrices.push_back(m);
    rep.rank_deficient.push_back(r.rank_deficient[k] != 0);
  }
  for (int c = 0; c < 3; ++c) {
    rep.threshold_m1[c] = r.threshold_m1[c];
    rep.threshold_m2[c] = r.threshold_m2[c];
  }
  ++state.frame_counter;
  return result;
}

struct RunResult {
  std::vector<Frame> panoramas;
  RunReport report;
};

// run_sequence (pipeline.hpp:90-92, pipeline.cpp:362-420); periodic
// re-refinement (refine.rerefine_every) runs through stitch_b200_rerefine.
inline RunResult run_sequence(const StitchConfig& config, const std::vector<std::vector<Frame>>& views,
                              const std::function<void(long, const Frame&)>& sink = {}) {
  if (views.size() != config.views.size())
    throw StitchError(ErrorCode::ConfigurationError, "stream count does not match configured views");
  const std::size_t frames = views.front().size();
  for (const auto& s : views)
    if (s.size() != frames)
      throw StitchError(ErrorCode::ConfigurationError, "streams must have equal length");
  if (frames == 0) throw StitchError(ErrorCode::ConfigurationError, "empty input streams");
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<Frame> first;
  for (const auto& s : views) first.push_back(s[0]);
  PipelineState state = initialize(config, first);
  RunResult result;
  result.report.scene_id = config.scene_id;
  result.report.threads = config.threads;
  result.report.frames = static_cast<long>(frames);
  // pipeline.cpp:390-392: any pair whose refinement fell back
  for (int k = 0; k < state.n_pairs(); ++k)
    result.report.refine_warning |= stitch_b200_refine_warning(state.handle(), k) != 0;
  const int every = config.refine.rerefine_every;
  for (std::size_t t = 0; t < frames; ++t) {
    std::vector<Frame> set;
    for (const auto& s : views) set.push_back(s[t]);
    if (every > 0 && t > 0 && t % static_cast<std::size_t>(every) == 0) {
      // re-refinement (pipeline.cpp:395-406): fresh initialize() on the
      // current frames, windows / history / counter carried over
      stitch_b200_config c = to_c(config, set);
      std::vector<const std::uint8_t*> ptrs;
      for (const Frame& f : set) ptrs.push_back(f.data.data());
      check(stitch_b200_rerefine(state.handle(), &c, ptrs.data()));
    }
    ProcessResult pr = process_frame(state, set);
    result.report.totals += pr.report.times;
    result.report.per_frame.push_back(pr.report);
    if (sink)
      sink(static_cast<long>(t), pr.panorama);
    else
      result.panoramas.push_back(std::move(pr.panorama));
  }
  result.report.wall_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return result;
}

// ---- image_io.hpp (image_io.cpp:61-199); PNG on zlib (no libpng here) ----
inline Frame read_ppm(const std::string& path) {
  int w = 0, h = 0;
  check(stitch_b200_read_ppm(path.c_str(), nullptr, 0, &w, &h));
  Frame f(w, h);
  check(stitch_b200_read_ppm(path.c_str(), f.data.data(), f.data.size(), nullptr, nullptr));
  return f;
}

inline void write_ppm(const std::string& path, const Frame& frame) {
  if (frame.data.size() != frame.pixel_count() * 3)
    throw StitchError(ErrorCode::InputMismatch, "frame data must be width*height*3 bytes");
  check(stitch_b200_write_ppm(path.c_str(), frame.width, frame.height, frame.data.data()));
}

inline Frame read_png(const std::string& path) {
  int w = 0, h = 0, hm = 0;
  check(stitch_b200_read_png(path.c_str(), nullptr, 0, nullptr, 0, &w, &h, &hm));
  Frame f(w, h);
  std::vector<std::uint8_t> mask(f.pixel_count());
  check(stitch_b200_read_png(path.c_str(), f.data.data(), f.data.size(), mask.data(), mask.size(),
                             nullptr, nullptr, nullptr));
  if (hm) f.mask = std::move(mask);
  return f;
}

inline void write_png(const std::string& path, const Frame& frame) {
  if (frame.data.size() != frame.pixel_count() * 3)
    throw StitchError(ErrorCode::InputMismatch, "frame data must be width*height*3 bytes");
  check(stitch_b200_write_png(path.c_str(), frame.width, frame.height, frame.data.data(),
                              frame.has_mask() ? frame.mask.data() : nullptr));
}

inline std::string sequence_name(const std::string& stem, int index,
                                 const std::string& ext = ".png") {
  std::vector<char> buf(stem.size() + ext.size() + 32);
  check(stitch_b200_sequence_name(stem.c_str(), index, ext.c_str(), buf.data(), buf.size()));
  return std::string(buf.data());
}

struct FilesRunResult {
  std::vector<FrameReport> per_frame;
  long frames = 0;
  double wall_seconds = 0.0, read_seconds = 0.0, write_seconds = 0.0;
  double fps() const { return wall_seconds > 0 ? frames / wall_seconds : 0.0; }
};

// run_sequence over numbered PPM sequences (one directory per view) with the
// panoramas written to out_dir/<stem>_%06d.ppm (empty out_dir: not written);
// reads, GPU frames and writes overlap inside the library.
inline FilesRunResult run_files(PipelineState& state, const std::vector<std::string>& view_dirs,
                                const std::string& out_dir = {}, const std::string& stem = "pano",
                                int max_frames = 0, const std::string& ext = ".ppm") {
  std::vector<const char*> dirs;
  for (const auto& d : view_dirs) dirs.push_back(d.c_str());
  if (static_cast<int>(dirs.size()) != stitch_b200_n_views(state.handle()))
    throw StitchError(ErrorCode::InputMismatch, "one directory per view");
  std::vector<stitch_b200_report> reps;
  stitch_b200_files_stats st{};
  // reports are collected only for a bounded run (max_frames > 0)
  if (max_frames > 0) reps.resize(static_cast<std::size_t>(max_frames));
  check(stitch_b200_run_files(state.handle(), dirs.data(), out_dir.empty() ? nullptr : out_dir.c_str(),
                              stem.c_str(), ext.c_str(), max_frames,
                              reps.empty() ? nullptr : reps.data(), &st));
  FilesRunResult res;
  res.frames = static_cast<long>(st.frames);
  res.wall_seconds = st.seconds;
  res.read_seconds = st.read_seconds;
  res.write_seconds = st.write_seconds;
  for (long t = 0; t < res.frames && !reps.empty(); ++t) {
    const stitch_b200_report& r = reps[static_cast<std::size_t>(t)];
    FrameReport rep;
    rep.frame_index = static_cast<long>(r.frame_index);
    for (int i = 0; i < kStageCount; ++i) rep.times.seconds[i] = r.stage_ms[i] * 1e-3;
    for (int k = 0; k < r.n_pairs; ++k) {
      Matrix3d m;
      for (int i = 0; i < 9; ++i) m[i] = r.color_matrices[k][i];
      rep.color_matrices.push_back(m);
      rep.rank_deficient.push_back(r.rank_deficient[k] != 0);
    }
    for (int c = 0; c < 3; ++c) {
      rep.threshold_m1[c] = r.threshold_m1[c];
      rep.threshold_m2[c] = r.threshold_m2[c];
    }
    res.per_frame.push_back(rep);
  }
  state.frame_counter += res.frames;
  return res;
}

}  // namespace stitch_b200
