// TEST INFRASTRUCTURE ONLY -- C ABI over the UNMODIFIED reference sources.
//
// oracle/ref/Makefile compiles /root/reference/proj/src/{frame,histogram,
// geometry,color_transfer,color_balance,flow,pipeline,parallel,features,
// integral,synth,config}.cpp where they lie (no copies), against the
// Eigen-subset shim in oracle/ref/eigen_shim, and links them with this file
// into oracle/_ref/libstitch_ref.so.  Nothing here re-implements the
// algorithm: every entry point forwards to the reference's own public API
// (pipeline.hpp:73-92, synth.hpp:47-92, color_balance.hpp:38-52) so that
// tests/test_ref_pin.py can pin oracle/stitch_oracle.c -- and through it the
// B200 path -- to the reference's own outputs.  Only tests/ and bench.py's
// `--impl reference` arm load the library; the product never does.
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <vector>

#include "stitch/color_balance.hpp"
#include "stitch/pipeline.hpp"
#include "stitch/synth.hpp"
#include "stitch/types.hpp"

namespace {

constexpr int kMax = 16;
thread_local char g_err[512];

int fail(const std::exception& e) {
  std::snprintf(g_err, sizeof(g_err), "%s", e.what());
  if (auto* se = dynamic_cast<const stitch::StitchError*>(&e))
    return static_cast<int>(se->code());
  return 1000;
}

struct Scene {
  stitch::SynthScene scene;
};

struct State {
  stitch::PipelineState st;
  stitch::FrameReport last;
};

}  // namespace

extern "C" {

// Mirrors stitch::SynthSpec (synth.hpp:31-44) as a POD.
struct ref_spec {
  uint64_t seed;
  int views, frames, width, height;
  double overlap_fraction;
  int n_casts;
  double casts[kMax][3];
  int n_flicker;
  struct {
    int frame, view;
    double gains[3];
  } flicker[kMax];
  int object_enabled;
  double depth_fraction, half_size, position[2], velocity[2];
  double perturb_focal_scale, perturb_principal_px;
};

// The StitchConfig fields a test may override (pipeline.hpp:17-45);
// everything else keeps SynthScene::config() (synth.cpp:156-179).
struct ref_opts {
  double lambda, gamma_dark, gamma_bright;
  int target_black, target_white;
  int levels, iterations;
  double smoothness;
  int window_capacity, fuse_weighting, threads;
  int refine_enabled;
  double refine_margin;
  int ransac_iters;
  double inlier_px, detect_threshold, match_ratio;
  int rerefine_every;
};

struct ref_report {
  long frame_index;
  int n_pairs;
  double m[kMax][9];  // row-major color_matrices
  int rank_deficient[kMax];
  int m1[3], m2[3];
};

const char* ref_last_error() { return g_err; }

void ref_default_opts(ref_opts* o) {
  const stitch::StitchConfig c;
  o->lambda = c.balance.lambda;
  o->gamma_dark = c.balance.gamma_dark;
  o->gamma_bright = c.balance.gamma_bright;
  o->target_black = c.balance.target_black;
  o->target_white = c.balance.target_white;
  o->levels = c.flow.levels;
  o->iterations = c.flow.iterations;
  o->smoothness = c.flow.smoothness;
  o->window_capacity = c.window_capacity;
  o->fuse_weighting = static_cast<int>(c.fuse_weighting);
  o->threads = c.threads;
  o->refine_enabled = c.refine.enabled ? 1 : 0;
  o->refine_margin = c.refine.margin;
  o->ransac_iters = c.refine.ransac_iters;
  o->inlier_px = c.refine.inlier_px;
  o->detect_threshold = c.refine.detect_threshold;
  o->match_ratio = c.refine.match_ratio;
  o->rerefine_every = c.refine.rerefine_every;
}

void* ref_scene_new(const ref_spec* s, int* err) {
  try {
    stitch::SynthSpec spec;
    spec.seed = s->seed;
    spec.views = s->views;
    spec.frames = s->frames;
    spec.width = s->width;
    spec.height = s->height;
    spec.overlap_fraction = s->overlap_fraction;
    for (int v = 0; v < s->n_casts; ++v)
      spec.color_casts.push_back({s->casts[v][0], s->casts[v][1], s->casts[v][2]});
    for (int i = 0; i < s->n_flicker; ++i) {
      stitch::FlickerEvent f;
      f.frame = s->flicker[i].frame;
      f.view = s->flicker[i].view;
      f.gains = {s->flicker[i].gains[0], s->flicker[i].gains[1], s->flicker[i].gains[2]};
      spec.flicker.push_back(f);
    }
    spec.object.enabled = s->object_enabled != 0;
    spec.object.depth_fraction = s->depth_fraction;
    spec.object.half_size = s->half_size;
    spec.object.position = Eigen::Vector2d(s->position[0], s->position[1]);
    spec.object.velocity = Eigen::Vector2d(s->velocity[0], s->velocity[1]);
    spec.perturb_focal_scale = s->perturb_focal_scale;
    spec.perturb_principal_px = s->perturb_principal_px;
    auto* sc = new Scene{stitch::synth_scene(spec)};
    *err = -1;
    return sc;
  } catch (const std::exception& e) {
    *err = fail(e);
    return nullptr;
  }
}

void ref_scene_free(void* p) { delete static_cast<Scene*>(p); }

int ref_scene_reference(void* p) { return static_cast<Scene*>(p)->scene.reference_view(); }

// RGB8 of view v at frame t (synth.cpp:181-231), W*H*3 bytes.
int ref_scene_render(void* p, int view, int frame, uint8_t* rgb) {
  try {
    const stitch::Frame f = static_cast<Scene*>(p)->scene.render_view(view, frame);
    std::memcpy(rgb, f.data.data(), f.data.size());
    return -1;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Per view (pipeline config, perturbation applied): fx fy cx cy R[9] t[3].
int ref_scene_cameras(void* p, double* out) {
  const stitch::StitchConfig c = static_cast<Scene*>(p)->scene.config();
  for (std::size_t v = 0; v < c.views.size(); ++v) {
    double* o = out + 16 * v;
    const auto& in = c.views[v].intrinsics;
    const auto& ex = c.views[v].extrinsics;
    o[0] = in.fx;
    o[1] = in.fy;
    o[2] = in.cx;
    o[3] = in.cy;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) o[4 + 3 * i + j] = ex.rotation(i, j);
    for (int i = 0; i < 3; ++i) o[13 + i] = ex.translation(i);
  }
  return static_cast<int>(c.views.size());
}

static stitch::StitchConfig make_config(const Scene* sc, const ref_opts* o) {
  stitch::StitchConfig c = sc->scene.config();
  c.balance.lambda = o->lambda;
  c.balance.gamma_dark = o->gamma_dark;
  c.balance.gamma_bright = o->gamma_bright;
  c.balance.target_black = o->target_black;
  c.balance.target_white = o->target_white;
  c.flow.levels = o->levels;
  c.flow.iterations = o->iterations;
  c.flow.smoothness = o->smoothness;
  c.flow.threads = o->threads;
  c.window_capacity = o->window_capacity;
  c.fuse_weighting = static_cast<stitch::FuseWeighting>(o->fuse_weighting);
  c.threads = o->threads;
  c.refine.enabled = o->refine_enabled != 0;
  c.refine.margin = o->refine_margin;
  c.refine.ransac_iters = o->ransac_iters;
  c.refine.inlier_px = o->inlier_px;
  c.refine.detect_threshold = o->detect_threshold;
  c.refine.match_ratio = o->match_ratio;
  c.refine.rerefine_every = o->rerefine_every;
  return c;
}

// masks: NULL, or per view NULL (no mask) or width*height 0/1 bytes
static std::vector<stitch::Frame> wrap(const std::vector<std::pair<int, int>>& sizes,
                                       const uint8_t* const* rgb,
                                       const uint8_t* const* masks = nullptr) {
  std::vector<stitch::Frame> out;
  for (std::size_t v = 0; v < sizes.size(); ++v) {
    stitch::Frame f(sizes[v].first, sizes[v].second);
    std::memcpy(f.data.data(), rgb[v], f.data.size());
    if (masks && masks[v]) f.mask.assign(masks[v], masks[v] + f.pixel_count());
    out.push_back(std::move(f));
  }
  return out;
}

static std::vector<std::pair<int, int>> scene_sizes(const Scene* sc) {
  const auto& s = sc->scene.spec();
  return std::vector<std::pair<int, int>>(static_cast<std::size_t>(s.views),
                                          {s.width, s.height});
}

// stitch::initialize (pipeline.cpp:209-257) on caller-supplied first frames.
void* ref_state_new(void* scene, const ref_opts* o, const uint8_t* const* first,
                    const uint8_t* const* first_masks, int* err) {
  try {
    const auto* sc = static_cast<Scene*>(scene);
    auto* st = new State;
    st->st = stitch::initialize(make_config(sc, o), wrap(scene_sizes(sc), first, first_masks));
    *err = -1;
    return st;
  } catch (const std::exception& e) {
    *err = fail(e);
    return nullptr;
  }
}

void ref_state_free(void* p) { delete static_cast<State*>(p); }

void ref_state_canvas(void* p, int* w, int* h, double* ox, double* oy) {
  const auto& c = static_cast<State*>(p)->st.canvas;
  *w = c.width;
  *h = c.height;
  *ox = c.offset.x();
  *oy = c.offset.y();
}

// warp_maps[v].h (row-major) and the raw Eigen inverse process_frame warps with
// (pipeline.cpp:40).
void ref_state_map(void* p, int v, double* h9, double* inv9) {
  const auto& m = static_cast<State*>(p)->st.warp_maps[static_cast<std::size_t>(v)].h;
  const Eigen::Matrix3d inv = m.inverse();
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      h9[3 * i + j] = m(i, j);
      inv9[3 * i + j] = inv(i, j);
    }
}

int ref_state_n_pairs(void* p) { return static_cast<int>(static_cast<State*>(p)->st.pairs.size()); }

void ref_state_pair(void* p, int k, int* view, int* bounds, int* refine_warning) {
  const auto& pr = static_cast<State*>(p)->st.pairs[static_cast<std::size_t>(k)];
  *view = pr.view;
  bounds[0] = pr.bounds.x0;
  bounds[1] = pr.bounds.y0;
  bounds[2] = pr.bounds.x1;
  bounds[3] = pr.bounds.y1;
  *refine_warning = pr.refine_warning ? 1 : 0;
}

void ref_state_pair_weights(void* p, int k, float* theta_i, float* theta_j) {
  const auto& w = static_cast<State*>(p)->st.pairs[static_cast<std::size_t>(k)].weights;
  for (int y = 0; y < w.height; ++y)
    for (int x = 0; x < w.width; ++x) {
      theta_i[static_cast<std::size_t>(y) * w.width + x] = w.theta_i(y, x);
      theta_j[static_cast<std::size_t>(y) * w.width + x] = w.theta_j(y, x);
    }
}

// stitch::process_frame (pipeline.cpp:259-360) on n frames of the given sizes.
// pano_rgb: canvas W*H*3; pano_mask: canvas W*H (all ones when the reference
// returns no mask).
int ref_process_sized(void* p, int n, const int* widths, const int* heights,
                      const uint8_t* const* frames, const uint8_t* const* masks,
                      uint8_t* pano_rgb, uint8_t* pano_mask, ref_report* rep) {
  try {
    auto* st = static_cast<State*>(p);
    std::vector<std::pair<int, int>> sizes;
    for (int v = 0; v < n; ++v) sizes.emplace_back(widths[v], heights[v]);
    stitch::ProcessResult r = stitch::process_frame(st->st, wrap(sizes, frames, masks));
    const stitch::Frame& pano = r.panorama;
    std::memcpy(pano_rgb, pano.data.data(), pano.data.size());
    if (pano.has_mask())
      std::memcpy(pano_mask, pano.mask.data(), pano.mask.size());
    else
      std::memset(pano_mask, 1, pano.pixel_count());
    rep->frame_index = r.report.frame_index;
    rep->n_pairs = static_cast<int>(r.report.color_matrices.size());
    for (int k = 0; k < rep->n_pairs && k < kMax; ++k) {
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) rep->m[k][3 * i + j] = r.report.color_matrices[k](i, j);
      rep->rank_deficient[k] = r.report.rank_deficient[k] ? 1 : 0;
    }
    for (int c = 0; c < 3; ++c) {
      rep->m1[c] = r.report.threshold_m1[c];
      rep->m2[c] = r.report.threshold_m2[c];
    }
    return -1;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

static stitch::Frame frame_of(int w, int h, const uint8_t* rgb, const uint8_t* mask) {
  stitch::Frame f(w, h);
  std::memcpy(f.data.data(), rgb, f.data.size());
  if (mask) f.mask.assign(mask, mask + f.pixel_count());
  return f;
}

// dense_flow (flow.cpp:140-187) from a to b (equal sizes; masks optional).
int ref_dense_flow(int w, int h, const uint8_t* a_rgb, const uint8_t* a_mask,
                   const uint8_t* b_rgb, const uint8_t* b_mask, int levels, int iterations,
                   double smoothness, int threads, float* u, float* v) {
  try {
    stitch::FlowOptions o;
    o.levels = levels;
    o.iterations = iterations;
    o.smoothness = smoothness;
    o.threads = threads;
    const stitch::FlowField f =
        stitch::dense_flow(frame_of(w, h, a_rgb, a_mask), frame_of(w, h, b_rgb, b_mask), o);
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) {
        u[static_cast<std::size_t>(y) * w + x] = f.u(y, x);
        v[static_cast<std::size_t>(y) * w + x] = f.v(y, x);
      }
    return -1;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// warp_frame (geometry.cpp:58-83) of a w x h frame through the homography h9
// (row-major, taken as is) onto a cw x ch canvas at offset (ox, oy).
int ref_warp_frame(int w, int h, const uint8_t* rgb, const uint8_t* mask, const double* h9,
                   int cw, int ch, double ox, double oy, uint8_t* out_rgb, uint8_t* out_mask) {
  try {
    stitch::Homography hm;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) hm.h(i, j) = h9[3 * i + j];
    const stitch::Frame f =
        stitch::warp_frame(frame_of(w, h, rgb, mask), hm, cw, ch, Eigen::Vector2d(ox, oy));
    std::memcpy(out_rgb, f.data.data(), f.data.size());
    if (f.has_mask())
      std::memcpy(out_mask, f.mask.data(), f.mask.size());
    else
      std::memset(out_mask, 1, f.pixel_count());
    return -1;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// build_curve (color_balance.cpp:65-104) -> 3x256 LUT.
void ref_build_curve(const int* m1, const int* m2, double gamma_dark, double gamma_bright,
                     int target_black, int target_white, uint8_t* out) {
  stitch::BalanceThresholds th;
  for (int c = 0; c < 3; ++c) {
    th.m1[c] = m1[c];
    th.m2[c] = m2[c];
  }
  stitch::BalanceConfig cfg;
  cfg.gamma_dark = gamma_dark;
  cfg.gamma_bright = gamma_bright;
  cfg.target_black = target_black;
  cfg.target_white = target_white;
  const stitch::ToneLUT lut = stitch::build_curve(th, cfg);
  for (int c = 0; c < 3; ++c)
    for (int v = 0; v < 256; ++v) out[256 * c + v] = lut.map[c][v];
}

}  // extern "C"
