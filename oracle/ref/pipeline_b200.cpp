// The reference-side binding a maintainer adds, compiled
// here against the reference's own headers (/root/reference/proj/include) by
// oracle/ref/Makefile so that it is known to build and -- through
// oracle/ref/integration_demo.cpp -- to reproduce stitch::process_frame.
//
// process_frame_b200 is a drop-in for process_frame (pipeline.hpp:79-80):
// same inputs, same ProcessResult, same exceptions.  The device twin of a
// PipelineState (a stitch_b200 context) lives in a side table keyed by the
// state's address; release_b200 destroys it.  The table also stores a
// fingerprint of the geometry the twin was built from, so a state whose
// geometry changed under the same address is caught: a fresh state
// (frame_counter == 0) gets a fresh twin, a re-refined one (run_sequence's
// rerefine branch, pipeline.cpp:395-406: windows, history and counter
// carried over) gets stitch_b200_update_geometry, which keeps the device's
// temporal state exactly as the reference carries it.
#include <cstring>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "stitch/pipeline.hpp"
#include "stitch_b200.h"

namespace stitch {

namespace {

void throw_b200(int status) {
  if (status == STITCH_B200_OK) return;
  const auto code = (status >= 1 && status <= 17) ? static_cast<ErrorCode>(status - 1)
                                                  : ErrorCode::ConfigurationError;
  throw StitchError(code, stitch_b200_last_error());
}

// The values process_frame reads from the state, as a stitch_b200_init
// (theta pointers borrow the state's PlaneF storage until create returns).
stitch_b200_init snapshot(const PipelineState& s, const std::vector<Frame>& frames) {
  stitch_b200_init in{};
  in.canvas_width = s.canvas.width;
  in.canvas_height = s.canvas.height;
  in.canvas_offset[0] = s.canvas.offset.x();
  in.canvas_offset[1] = s.canvas.offset.y();
  in.n_views = static_cast<int>(s.warp_maps.size());
  in.reference = s.config.reference;
  for (int v = 0; v < in.n_views; ++v) {
    in.view_width[v] = frames[v].width;
    in.view_height[v] = frames[v].height;
    const Eigen::Matrix3d inv = s.warp_maps[v].h.inverse();  // as pipeline.cpp:40
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) in.inv_maps[v][r * 3 + c] = inv(r, c);
  }
  in.n_pairs = static_cast<int>(s.pairs.size());
  for (int k = 0; k < in.n_pairs; ++k) {
    const auto& p = s.pairs[k];
    in.pairs[k].view = p.view;
    in.pairs[k].partner = s.config.reference;  // star: every pair against the reference
    in.pairs[k].x0 = p.bounds.x0;
    in.pairs[k].y0 = p.bounds.y0;
    in.pairs[k].x1 = p.bounds.x1;
    in.pairs[k].y1 = p.bounds.y1;
    in.pairs[k].theta_i = p.weights.theta_i.data();  // row-major PlaneF
  }
  in.window_capacity = s.config.window_capacity;
  in.lambda = s.config.balance.lambda;
  in.gamma_dark = s.config.balance.gamma_dark;
  in.gamma_bright = s.config.balance.gamma_bright;
  in.target_black = s.config.balance.target_black;
  in.target_white = s.config.balance.target_white;
  in.flow_levels = s.config.flow.levels;
  in.flow_iterations = s.config.flow.iterations;
  in.smoothness = s.config.flow.smoothness;
  in.fuse_weighting = s.config.fuse_weighting == FuseWeighting::CrossWeightOnOwnFlow ? 1 : 0;
  return in;
}

// What the twin was built from: canvas, maps, pair bounds.
std::vector<double> fingerprint(const PipelineState& s) {
  std::vector<double> f{static_cast<double>(s.canvas.width), static_cast<double>(s.canvas.height),
                        s.canvas.offset.x(), s.canvas.offset.y()};
  for (const auto& m : s.warp_maps)
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) f.push_back(m.h(r, c));
  for (const auto& p : s.pairs) {
    f.push_back(p.view);
    f.push_back(p.bounds.x0);
    f.push_back(p.bounds.y0);
    f.push_back(p.bounds.x1);
    f.push_back(p.bounds.y1);
  }
  return f;
}

struct Twin {
  stitch_b200_ctx* ctx = nullptr;
  std::vector<double> built_from;
  ~Twin() {
    if (ctx) stitch_b200_destroy(ctx);
  }
};

std::mutex g_mu;
std::unordered_map<const PipelineState*, std::unique_ptr<Twin>> g_twins;

}  // namespace

// Drop-in for process_frame (pipeline.cpp:259-360) on the GPU.
ProcessResult process_frame_b200(PipelineState& state, const std::vector<Frame>& frames,
                                 int device = 0) {
  if (frames.size() != state.config.views.size())
    throw StitchError(ErrorCode::ConfigurationError, "frame count does not match configured views");
  Twin* twin;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto& slot = g_twins[&state];
    const std::vector<double> fp = fingerprint(state);
    if (slot && slot->built_from != fp) {
      if (state.frame_counter == 0) {
        slot.reset();  // a new pipeline at the same address
      } else {         // re-refined geometry, temporal state carried over
        const stitch_b200_init in = snapshot(state, frames);
        throw_b200(stitch_b200_update_geometry(slot->ctx, &in));
        slot->built_from = fp;
      }
    }
    if (!slot) {
      slot = std::make_unique<Twin>();
      const stitch_b200_init in = snapshot(state, frames);
      throw_b200(stitch_b200_create(&in, device, &slot->ctx));
      slot->built_from = fp;
    }
    twin = slot.get();
  }
  std::vector<const uint8_t*> ptrs, masks;
  std::vector<int> ws, hs;
  for (const Frame& f : frames) {
    ptrs.push_back(f.data.data());
    masks.push_back(f.has_mask() ? f.mask.data() : nullptr);
    ws.push_back(f.width);
    hs.push_back(f.height);
  }
  // sizes as the twin was built for
  throw_b200(stitch_b200_check_frames(twin->ctx, static_cast<int>(frames.size()), ws.data(),
                                      hs.data(), masks.data()));
  bool any_mask = false;
  for (const uint8_t* m : masks) any_mask = any_mask || m != nullptr;
  int cw = 0, ch = 0;
  throw_b200(stitch_b200_canvas(twin->ctx, &cw, &ch, nullptr, nullptr));
  ProcessResult result;
  result.panorama = Frame::with_mask(cw, ch, 0, 0);
  stitch_b200_report r;
  if (any_mask)  // Frame::mask (frame.hpp:44-47): masked taps drop out (frame.cpp:95-104)
    throw_b200(stitch_b200_process_masked(twin->ctx, ptrs.data(), masks.data(),
                                          result.panorama.data.data(),
                                          result.panorama.mask.data(), &r));
  else
    throw_b200(stitch_b200_process(twin->ctx, ptrs.data(), result.panorama.data.data(),
                                   result.panorama.mask.data(), &r));
  result.report.frame_index = state.frame_counter++;
  for (int k = 0; k < r.n_pairs; ++k) {
    Eigen::Matrix3d m;
    for (int i = 0; i < 9; ++i) m(i / 3, i % 3) = r.color_matrices[k][i];
    result.report.color_matrices.push_back(m);
    result.report.rank_deficient.push_back(r.rank_deficient[k] != 0);
  }
  for (int c = 0; c < 3; ++c) {
    result.report.threshold_m1[c] = r.threshold_m1[c];
    result.report.threshold_m2[c] = r.threshold_m2[c];
  }
  for (int i = 0; i < kStageCount; ++i) result.report.times.seconds[i] = r.stage_ms[i] * 1e-3;
  return result;
}

// Destroys the device twin of `state` (call before the state goes away).
void release_b200(const PipelineState& state) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_twins.erase(&state);
}

}  // namespace stitch
