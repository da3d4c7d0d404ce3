// TEST INFRASTRUCTURE: the drop-in, end to end.  The reference itself
// (unmodified sources, oracle/_ref) renders a synthetic rig and runs
// stitch::initialize; a copy of the resulting PipelineState is then driven
// frame by frame through both stitch::process_frame (the reference, CPU) and
// the maintainer's binding process_frame_b200 (oracle/ref/pipeline_b200.cpp
// -> libstitch_b200.so on the GPU), and every output is compared byte for
// byte: panorama RGB and mask, colour matrices (bitwise), rank flags,
// thresholds, frame index.  Prints one JSON line; exit 0 iff identical.
//
//   integration_demo <views> <width> <height> <frames> [refine 0|1] [device] [masked 0|1|2]
//
// masked = 1 gives every view a per-frame Frame::mask (a moving hole, a cut
// border strip, scattered pixels), first frames included, as a PNG source
// with alpha would (image_io.cpp:120-127).  masked = 2 also masks frame 2 of
// the last view completely: the reference throws EmptyProjection there
// (geometry.cpp:79) and the binding must throw the same code, with both
// states left untouched for the frames after it.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "stitch/pipeline.hpp"
#include "stitch/synth.hpp"

namespace stitch {
ProcessResult process_frame_b200(PipelineState& state, const std::vector<Frame>& frames,
                                 int device);
void release_b200(const PipelineState& state);
}  // namespace stitch

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: %s views width height frames [refine] [device]\n", argv[0]);
    return 2;
  }
  stitch::SynthSpec spec;
  spec.seed = 1;
  spec.views = std::atoi(argv[1]);
  spec.width = std::atoi(argv[2]);
  spec.height = std::atoi(argv[3]);
  spec.frames = std::atoi(argv[4]);
  const bool refine = argc > 5 ? std::atoi(argv[5]) != 0 : true;
  const int device = argc > 6 ? std::atoi(argv[6]) : 0;
  const int masked_mode = argc > 7 ? std::atoi(argv[7]) : 0;
  const bool masked = masked_mode != 0;
  auto add_mask = [&](stitch::Frame& f, int view, int t) {
    if (!masked) return;
    if (masked_mode == 2 && t == 2 && view == spec.views - 1) {
      f.mask.assign(f.pixel_count(), 0);  // nothing valid: EmptyProjection
      return;
    }
    f.mask.assign(f.pixel_count(), 1);
    const int cx = (f.width / 3 + 9 * t + 31 * view) % f.width;
    const int cy = (f.height / 2 + 5 * t) % f.height;
    const int r = std::max(3, f.height / 9);
    for (int y = 0; y < f.height; ++y)
      for (int x = 0; x < f.width; ++x) {
        const bool hole = (x - cx) * (x - cx) + (y - cy) * (y - cy) <= r * r;
        const bool strip = view % 2 ? x >= f.width - 4 : x < 4;
        const bool dot = ((x * 7 + y * 13 + t * 3 + view) % 89) == 0;
        if (hole || strip || dot) f.mask[f.index(x, y)] = 0;
      }
  };
  spec.overlap_fraction = 0.3;
  for (int v = 0; v < spec.views; ++v)
    spec.color_casts.push_back(v == 0 ? std::array<double, 3>{1, 1, 1}
                                      : std::array<double, 3>{0.85 + 0.05 * v, 1.0, 1.1 - 0.05 * v});
  spec.flicker.push_back({3, spec.views - 1, {1.25, 1.1, 0.9}});
  spec.object.enabled = true;
  spec.object.half_size = 40.0;
  spec.object.velocity = Eigen::Vector2d(3.0, 1.0);
  const stitch::SynthScene scene = stitch::synth_scene(spec);
  stitch::StitchConfig cfg = scene.config();
  cfg.refine.enabled = refine;
  cfg.threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  cfg.flow.threads = cfg.threads;
  std::vector<stitch::Frame> first;
  for (int v = 0; v < spec.views; ++v) {
    first.push_back(scene.render_view(v, 0));
    add_mask(first.back(), v, 0);
  }
  stitch::PipelineState cpu = stitch::initialize(cfg, first);
  stitch::PipelineState gpu = cpu;  // the same initialized state, driven by the binding
  int differing = 0, max_diff = 0, errors = 0;
  bool masks = true, reports = true, errors_equal = true;
  for (int t = 0; t < spec.frames; ++t) {
    std::vector<stitch::Frame> frames;
    for (int v = 0; v < spec.views; ++v) {
      frames.push_back(scene.render_view(v, t));
      add_mask(frames.back(), v, t);
    }
    stitch::ProcessResult a, b;
    int ea = -1, eb = -1;
    try {
      a = stitch::process_frame(cpu, frames);
    } catch (const stitch::StitchError& e) {
      ea = static_cast<int>(e.code());
    }
    try {
      b = stitch::process_frame_b200(gpu, frames, device);
    } catch (const stitch::StitchError& e) {
      eb = static_cast<int>(e.code());
    } catch (const std::exception& e) {
      std::printf("{\"error\": \"%s\"}\n", e.what());
      return 1;
    }
    if (ea != eb) errors_equal = false;
    if (ea >= 0 || eb >= 0) {  // both threw (or a mismatch, already counted)
      errors += ea >= 0;
      continue;
    }
    const std::vector<std::uint8_t> am =
        a.panorama.has_mask() ? a.panorama.mask
                              : std::vector<std::uint8_t>(a.panorama.pixel_count(), 1);
    masks = masks && am == b.panorama.mask;
    int d = 0;
    for (std::size_t i = 0; i < a.panorama.data.size() && i < b.panorama.data.size(); ++i)
      d = std::max(d, std::abs(int(a.panorama.data[i]) - int(b.panorama.data[i])));
    if (a.panorama.data.size() != b.panorama.data.size()) d = 256;
    max_diff = std::max(max_diff, d);
    differing += d != 0;
    bool rep = a.report.frame_index == b.report.frame_index &&
               a.report.threshold_m1 == b.report.threshold_m1 &&
               a.report.threshold_m2 == b.report.threshold_m2 &&
               a.report.rank_deficient == b.report.rank_deficient &&
               a.report.color_matrices.size() == b.report.color_matrices.size();
    for (std::size_t k = 0; rep && k < a.report.color_matrices.size(); ++k)
      rep = std::memcmp(a.report.color_matrices[k].data(), b.report.color_matrices[k].data(),
                        9 * sizeof(double)) == 0;
    reports = reports && rep;
  }
  stitch::release_b200(gpu);
  const bool ok = differing == 0 && masks && reports && errors_equal;
  std::printf("{\"views\": %d, \"width\": %d, \"height\": %d, \"frames\": %d, \"refine\": %d, "
              "\"masked\": %d, "
              "\"canvas\": [%d, %d], \"frames_differing\": %d, \"max_abs_diff\": %d, "
              "\"masks_equal\": %s, \"reports_equal\": %s, \"errors\": %d, "
              "\"errors_equal\": %s, \"identical\": %s}\n",
              spec.views, spec.width, spec.height, spec.frames, refine ? 1 : 0, masked_mode,
              cpu.canvas.width,
              cpu.canvas.height, differing, max_diff, masks ? "true" : "false",
              reports ? "true" : "false", errors, errors_equal ? "true" : "false",
              ok ? "true" : "false");
  return ok ? 0 : 1;
}
