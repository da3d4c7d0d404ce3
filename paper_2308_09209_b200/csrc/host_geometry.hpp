// host_geometry.hpp -- init-time geometry on the host (runs once per
// context, not per frame).  Restates the reference's init path
// (/root/reference/proj/src/geometry.cpp:8-171, pipeline.cpp:209-257,
// flow.cpp:192-280) in plain C++; 3x3 products use a fixed left-to-right
// summation order and the 3x3 inverse follows Eigen's cofactor formula
// (Eigen/src/LU/InverseImpl.h), which pipeline.cpp:40 relies on.
#pragma once

#include <array>
#include <cstdint>
#include <cstring>
#include <vector>

#include "stitch_b200.h"

namespace stitch_b200_host {

// StitchConfig defaults of the reference (pipeline.hpp:23-44,
// color_balance.hpp:19-25, flow.hpp:29-34): stitch_b200_config_defaults and
// the synthetic scenes' configs (libstitch_synth.so) share this one copy.
inline void config_defaults(stitch_b200_config* c) {
  std::memset(c, 0, sizeof(*c));
  c->n_views = 2;
  c->reference = 0;
  c->lambda = 0.05;
  c->gamma_dark = 1.5;
  c->gamma_bright = 1.5;
  c->target_black = 0;
  c->target_white = 255;
  c->flow_levels = 4;
  c->flow_iterations = 50;
  c->smoothness = 15.0;
  c->window_capacity = 3;
  c->fuse_weighting = 0;
  c->topology = 0;
  c->refine_enabled = 1;  // RefineOptions::enabled (pipeline.hpp:24)
  c->projection = 0;
  c->cyl_focal = 0.0;
  c->refine_margin = 0.15;  // RefineOptions defaults (pipeline.hpp:23-31)
  c->ransac_iters = 500;
  c->inlier_px = 2.0;
  c->detect_threshold = 2e-4;
  c->match_ratio = 0.8;
  c->seed = 0;
  for (int v = 0; v < STITCH_B200_MAX_VIEWS; ++v) {
    c->cams[v].fx = c->cams[v].fy = 1.0;
    c->cams[v].rotation[0] = c->cams[v].rotation[4] = c->cams[v].rotation[8] = 1.0;
  }
}


using Mat3 = std::array<double, 9>;  // row-major

void mul3(const Mat3& a, const Mat3& b, Mat3& out);
double det3(const Mat3& m);
void inverse3(const Mat3& m, Mat3& out);  // raw Eigen cofactor inverse
// Homography::from_matrix (geometry.cpp:16-26); returns status.
int homography_from_matrix(const Mat3& m, Mat3& out);
// Homography::inverse (geometry.cpp:29-31): normalised inverse.
int homography_inverse(const Mat3& h, Mat3& out);
// Homography::apply (geometry.cpp:33-36)
void homography_apply(const Mat3& h, double x, double y, double& ox, double& oy);
// planar_homography (geometry.cpp:38-51)
int planar_homography(const stitch_b200_camera& c, Mat3& out);
// pairwise_homography (geometry.cpp:53-56)
int pairwise_homography(const Mat3& hi, const Mat3& hj, Mat3& out);

struct Canvas {
  int width = 0, height = 0;
  double offx = 0, offy = 0;
};
// compute_canvas (geometry.cpp:147-171)
Canvas compute_canvas(const std::vector<Mat3>& maps, const std::vector<std::pair<int, int>>& sizes);

struct PairSpec {
  int view = 0, partner = 0;
};
// Star pairs (pipeline.cpp:233-239), the N-view chain extension, or the
// ring chain (topology 3: partner = ring neighbour toward the reference).
std::vector<PairSpec> build_pairs(int n_views, int reference, int topology);

// ---- cylindrical 360-degree canvas (extension) ----
// A_v = K_v R_v R_ref^T: reference-frame ray -> homogeneous pixel of view v.
void cylinder_maps(const stitch_b200_config& cfg, std::vector<Mat3>& maps);
// canvas covering 2*pi around the reference camera, height from the
// cameras' border rays; f = pixels per radian.
Canvas cylinder_canvas(const stitch_b200_config& cfg, double f);
// per-column sin/cos of t = (x + offx)/f and per-row h = (y + offy)/f
void lift_tables(const Canvas& c, double f, std::vector<double>& lsin, std::vector<double>& lcos,
                 std::vector<double>& lh);

// ---- feature refinement, host part (features.cpp:236-354, geometry.cpp) ----
struct MatchPt {
  double ax, ay, bx, by, distance;
};
struct ScaleShift {
  double s_x = 1.0, s_y = 1.0, t_x = 0.0, t_y = 0.0;
};
// ransac_scale_translation over (ax, ay) -> (bx, by): STITCH_B200_OK,
// InsufficientMatches or NoConsensus; the reference's std::mt19937_64 and
// std::uniform_int_distribution<std::size_t> stream.
int ransac_scale_translation(std::vector<MatchPt> m, int iterations, double inlier_px,
                             double min_scale, double max_scale, std::uint64_t seed,
                             ScaleShift& out);
// broaden (geometry.cpp:119-133)
void broaden(const int r[4], double margin, const int b[4], int out[4]);

// (overlap bounds, view footprints and blend weights are computed on the
// device: geometry_kernels.cu)

}  // namespace stitch_b200_host
