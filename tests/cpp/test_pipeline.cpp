// C++ parity test of the reference-signature API (include/stitch_b200.hpp)
// against the CPU oracle, written in the style of the reference's doctest
// suites (proj/tests/test_imaging.cpp).  Needs a B200; run by
// tests/test_cpp_api.py (gpu marker).
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../oracle/stitch_oracle.h"
#include "stitch_b200.hpp"
#include "stitch_synth.h"

static int g_failures = 0, g_checks = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    ++g_checks;                                                          \
    if (!(cond)) {                                                       \
      ++g_failures;                                                      \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                    \
  } while (0)
#define TEST_CASE(name) static void name()

using namespace stitch_b200;

static stitch_b200_synth* make_scene(int views, int w, int h) {
  stitch_b200_synth_spec spec;
  stitch_b200_synth_defaults(&spec);
  spec.views = views;
  spec.width = w;
  spec.height = h;
  spec.frames = 4;
  spec.n_casts = views;
  for (int v = 0; v < views; ++v) {
    spec.color_casts[v][0] = 1.0 - 0.05 * v;
    spec.color_casts[v][1] = 1.0;
    spec.color_casts[v][2] = 1.0 + 0.04 * v;
  }
  spec.object_enabled = 1;
  spec.object_velocity[0] = 3.0;
  stitch_b200_synth* s = nullptr;
  check(stitch_b200_synth_create(&spec, &s));
  return s;
}

static StitchConfig config_of(stitch_b200_synth* s, stitch_b200_config& c) {
  check(stitch_b200_synth_config(s, &c));
  StitchConfig cfg;
  CHECK(cfg.refine.enabled);  // the reference's default (pipeline.hpp:24)
  cfg.refine.enabled = false;  // these cases compare with the unrefined oracle
  cfg.reference = c.reference;
  for (int v = 0; v < c.n_views; ++v) {
    ViewSetup vs;
    vs.intrinsics = {c.cams[v].fx, c.cams[v].fy, c.cams[v].cx, c.cams[v].cy};
    for (int i = 0; i < 9; ++i) vs.extrinsics.rotation[i] = c.cams[v].rotation[i];
    for (int i = 0; i < 3; ++i) vs.extrinsics.translation[i] = c.cams[v].translation[i];
    cfg.views.push_back(vs);
  }
  return cfg;
}

static so_config oracle_config(const stitch_b200_config& c) {
  so_config o{};
  o.n_views = c.n_views;
  o.reference = c.reference;
  for (int v = 0; v < c.n_views; ++v) {
    o.width[v] = c.width[v];
    o.height[v] = c.height[v];
    o.cams[v].fx = c.cams[v].fx;
    o.cams[v].fy = c.cams[v].fy;
    o.cams[v].cx = c.cams[v].cx;
    o.cams[v].cy = c.cams[v].cy;
    for (int i = 0; i < 9; ++i) o.cams[v].rotation[i] = c.cams[v].rotation[i];
    for (int i = 0; i < 3; ++i) o.cams[v].translation[i] = c.cams[v].translation[i];
  }
  o.lambda = 0.05;
  o.gamma_dark = o.gamma_bright = 1.5;
  o.target_black = 0;
  o.target_white = 255;
  o.flow_levels = 4;
  o.flow_iterations = 50;
  o.smoothness = 15.0;
  o.window_capacity = 3;
  o.threads = 4;
  return o;
}

TEST_CASE(process_frame_matches_oracle) {
  for (int views : {2, 3}) {
    stitch_b200_synth* s = make_scene(views, 320, 240);
    stitch_b200_config c;
    StitchConfig cfg = config_of(s, c);
    std::vector<std::vector<Frame>> streams(views);
    for (int v = 0; v < views; ++v)
      for (int t = 0; t < 4; ++t) {
        Frame f(320, 240);
        check(stitch_b200_synth_render(s, v, t, f.data.data(), 4));
        streams[v].push_back(f);
      }
    std::vector<Frame> first;
    for (int v = 0; v < views; ++v) first.push_back(streams[v][0]);
    PipelineState state = initialize(cfg, first);
    so_config oc = oracle_config(c);
    int err = 0;
    so_state* os = so_initialize(&oc, &err);
    CHECK(os != nullptr);
    for (int t = 0; t < 4; ++t) {
      std::vector<Frame> set;
      std::vector<so_frame> oset;
      for (int v = 0; v < views; ++v) {
        set.push_back(streams[v][t]);
        oset.push_back(so_frame{320, 240, streams[v][t].data.data(), nullptr});
      }
      ProcessResult r = process_frame(state, set);
      so_frame pano{};
      so_report rep{};
      CHECK(so_process_frame(os, oset.data(), &pano, &rep) == SO_OK);
      CHECK(pano.width == r.panorama.width && pano.height == r.panorama.height);
      int maxdiff = 0;
      bool mask_same = true;
      for (std::size_t i = 0; i < r.panorama.pixel_count(); ++i) {
        mask_same = mask_same && (r.panorama.mask[i] != 0) == (pano.mask[i] != 0);
        for (int ch = 0; ch < 3; ++ch)
          maxdiff = std::max(maxdiff, std::abs(int(r.panorama.data[3 * i + ch]) - int(pano.data[3 * i + ch])));
      }
      CHECK(mask_same);
      CHECK(maxdiff == 0);
      CHECK(static_cast<int>(r.report.color_matrices.size()) == rep.n_pairs);
      for (int k = 0; k < rep.n_pairs; ++k)
        for (int i = 0; i < 9; ++i) CHECK(r.report.color_matrices[k][i] == rep.m[k][i]);
      for (int ch = 0; ch < 3; ++ch) {
        CHECK(r.report.threshold_m1[ch] == rep.threshold_m1[ch]);
        CHECK(r.report.threshold_m2[ch] == rep.threshold_m2[ch]);
      }
      so_free_frame(&pano);
    }
    so_destroy(os);
    stitch_b200_synth_destroy(s);
  }
}

TEST_CASE(errors_surface_as_stitch_error) {
  StitchConfig cfg;
  cfg.views.resize(1);
  bool threw = false;
  try {
    initialize(cfg, std::vector<Frame>(1, Frame(16, 16)));
  } catch (const StitchError& e) {
    threw = e.code() == ErrorCode::ConfigurationError;
  }
  CHECK(threw);
  stitch_b200_synth* s = make_scene(2, 64, 48);
  stitch_b200_config c;
  StitchConfig ok = config_of(s, c);
  // refinement on blank first frames: no keypoints, so every pair keeps its
  // unrefined map and carries the refine warning (pipeline.cpp:171-177)
  ok.refine.enabled = true;
  PipelineState st = initialize(ok, std::vector<Frame>(2, Frame(64, 48)));
  CHECK(st.n_pairs() == 1);
  CHECK(stitch_b200_refine_warning(st.handle(), 0) == 1);
  stitch_b200_synth_destroy(s);
}

TEST_CASE(run_sequence_reports_every_frame) {
  stitch_b200_synth* s = make_scene(2, 160, 120);
  stitch_b200_config c;
  StitchConfig cfg = config_of(s, c);
  std::vector<std::vector<Frame>> streams(2);
  for (int v = 0; v < 2; ++v)
    for (int t = 0; t < 3; ++t) {
      Frame f(160, 120);
      check(stitch_b200_synth_render(s, v, t, f.data.data(), 4));
      streams[v].push_back(f);
    }
  long seen = 0;
  RunResult r = run_sequence(cfg, streams, [&](long t, const Frame& p) {
    CHECK(t == seen);
    CHECK(p.width > 0);
    ++seen;
  });
  CHECK(seen == 3);
  CHECK(r.report.frames == 3);
  CHECK(r.report.per_frame.size() == 3);
  CHECK(r.panoramas.empty());
  stitch_b200_synth_destroy(s);
}

TEST_CASE(quality_metrics_match_oracle) {
  // metrics.cpp psnr / ssim through the C ABI (device) against the oracle
  const int w = 96, h = 64;
  std::vector<std::uint8_t> a(w * h * 3), b(w * h * 3), mb(w * h, 1);
  unsigned x = 12345;
  for (size_t i = 0; i < a.size(); ++i) {
    x = x * 1103515245u + 12345u;
    a[i] = static_cast<std::uint8_t>(x >> 24);
    b[i] = static_cast<std::uint8_t>((3 * a[i] + ((x >> 16) & 255)) / 4);
  }
  for (int y = 0; y < 20; ++y)
    for (int xx = 0; xx < 30; ++xx) mb[y * w + xx] = 0;
  so_frame fa{w, h, a.data(), nullptr}, fb{w, h, b.data(), mb.data()};
  double gp = 0, op = 0, gs = 0, os = 0;
  check(stitch_b200_psnr(w, h, a.data(), nullptr, b.data(), mb.data(), &gp));
  CHECK(so_psnr(&fa, &fb, &op) == SO_OK);
  CHECK(gp == op);
  check(stitch_b200_ssim(w, h, a.data(), nullptr, b.data(), mb.data(), &gs));
  CHECK(so_ssim(&fa, &fb, &os) == SO_OK);
  CHECK(gs == os);
  double same = 0;
  check(stitch_b200_psnr(w, h, a.data(), nullptr, a.data(), nullptr, &same));
  CHECK(std::isinf(same));
}

TEST_CASE(update_maps_keeps_geometry_for_unchanged_maps) {
  // re-refinement with the unrefined maps rebuilds the same device geometry
  stitch_b200_synth* s = make_scene(3, 160, 120);
  stitch_b200_config c;
  StitchConfig cfg = config_of(s, c);
  std::vector<Frame> first(3, Frame(160, 120));
  for (int v = 0; v < 3; ++v) check(stitch_b200_synth_render(s, v, 0, first[v].data.data(), 4));
  PipelineState st = initialize(cfg, first);
  stitch_b200_pair p0{};
  std::vector<float> th0(160 * 120 * 2), th1(160 * 120 * 2);
  check(stitch_b200_get_pair(st.handle(), 0, &p0, th0.data()));
  std::vector<double> maps(9 * 3);
  check(stitch_b200_camera_maps(&c, maps.data()));
  std::vector<std::array<double, 9>> m(3);
  for (int v = 0; v < 3; ++v)
    for (int i = 0; i < 9; ++i) m[v][i] = maps[9 * v + i];
  process_frame(st, first);
  st.update_maps(m);
  stitch_b200_pair p1{};
  check(stitch_b200_get_pair(st.handle(), 0, &p1, th1.data()));
  CHECK(p0.x0 == p1.x0 && p0.y0 == p1.y0 && p0.x1 == p1.x1 && p0.y1 == p1.y1);
  const size_t n = static_cast<size_t>(p0.x1 - p0.x0) * (p0.y1 - p0.y0);
  bool same = true;
  for (size_t i = 0; i < n; ++i) same = same && th0[i] == th1[i];
  CHECK(same);
  ProcessResult r = process_frame(st, first);
  CHECK(r.report.frame_index == 1);  // the temporal state was carried over
  stitch_b200_synth_destroy(s);
}

TEST_CASE(run_files_writes_the_process_frame_panoramas) {
  // image_io PPM sequences in, PPM panoramas out (run_files) == process_frame
  stitch_b200_synth* s = make_scene(2, 160, 120);
  stitch_b200_config c;
  StitchConfig cfg = config_of(s, c);
  char tmpl[] = "/tmp/stitch_b200_cpp_XXXXXX";
  const std::string root = mkdtemp(tmpl);
  std::vector<std::string> dirs;
  std::vector<std::vector<Frame>> frames(4);
  for (int v = 0; v < 2; ++v) {
    dirs.push_back(root + "/view" + std::to_string(v));
    CHECK(std::system(("mkdir -p " + dirs.back()).c_str()) == 0);
    for (int t = 0; t < 4; ++t) {
      Frame f(160, 120);
      check(stitch_b200_synth_render(s, v, t, f.data.data(), 4));
      write_ppm(dirs.back() + "/" + sequence_name("cam", t, ".ppm"), f);
      Frame back = read_ppm(dirs.back() + "/" + sequence_name("cam", t, ".ppm"));
      CHECK(back.width == 160 && back.height == 120 && back.data == f.data);
      frames[t].push_back(f);
    }
  }
  PipelineState a = initialize(cfg, frames[0]);
  FilesRunResult fr = run_files(a, dirs, root + "/out", "pano", 4);
  CHECK(fr.frames == 4);
  CHECK(fr.per_frame.size() == 4);
  PipelineState b = initialize(cfg, frames[0]);
  for (int t = 0; t < 4; ++t) {
    ProcessResult pr = process_frame(b, frames[t]);
    Frame got = read_ppm(root + "/out/" + sequence_name("pano", t, ".ppm"));
    CHECK(got.data == pr.panorama.data);
    CHECK(fr.per_frame[t].frame_index == t);
    CHECK(fr.per_frame[t].color_matrices == pr.report.color_matrices);
  }
  bool threw = false;
  try {
    read_ppm(root + "/missing.ppm");
  } catch (const StitchError& e) {
    threw = e.code() == ErrorCode::IoError;
  }
  CHECK(threw);
  CHECK(std::system(("rm -rf " + root).c_str()) == 0);
  stitch_b200_synth_destroy(s);
}

int main() {
  process_frame_matches_oracle();
  errors_surface_as_stitch_error();
  run_sequence_reports_every_frame();
  quality_metrics_match_oracle();
  update_maps_keeps_geometry_for_unchanged_maps();
  run_files_writes_the_process_frame_panoramas();
  std::printf("%d checks, %d failures\n", g_checks, g_failures);
  return g_failures ? 1 : 0;
}
