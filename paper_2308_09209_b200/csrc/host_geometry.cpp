// host_geometry.cpp -- init-time geometry (see host_geometry.hpp).
// Compiled with -ffp-contract=off so the double arithmetic is unfused.
#include "host_geometry.hpp"

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <limits>
#include <random>
#include <tuple>

namespace stitch_b200_host {

void mul3(const Mat3& a, const Mat3& b, Mat3& out) {
  Mat3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r[i * 3 + j] = (a[i * 3 + 0] * b[0 * 3 + j] + a[i * 3 + 1] * b[1 * 3 + j]) +
                     a[i * 3 + 2] * b[2 * 3 + j];
  out = r;
}

static inline double cof3(const Mat3& m, int i, int j) {
  const int i1 = (i + 1) % 3, i2 = (i + 2) % 3;
  const int j1 = (j + 1) % 3, j2 = (j + 2) % 3;
  return m[i1 * 3 + j1] * m[i2 * 3 + j2] - m[i1 * 3 + j2] * m[i2 * 3 + j1];
}

double det3(const Mat3& m) {
  const double c0 = cof3(m, 0, 0), c1 = cof3(m, 1, 0), c2 = cof3(m, 2, 0);
  return (c0 * m[0] + c1 * m[3]) + c2 * m[6];
}

// Eigen compute_inverse<MatrixType, ResultType, 3>::run
void inverse3(const Mat3& m, Mat3& out) {
  const double c0 = cof3(m, 0, 0), c1 = cof3(m, 1, 0), c2 = cof3(m, 2, 0);
  const double det = (c0 * m[0] + c1 * m[3]) + c2 * m[6];
  const double invdet = 1.0 / det;
  Mat3 r;
  r[1 * 3 + 0] = cof3(m, 0, 1) * invdet;
  r[1 * 3 + 1] = cof3(m, 1, 1) * invdet;
  r[2 * 3 + 0] = cof3(m, 0, 2) * invdet;
  r[1 * 3 + 2] = cof3(m, 2, 1) * invdet;
  r[2 * 3 + 1] = cof3(m, 1, 2) * invdet;
  r[2 * 3 + 2] = cof3(m, 2, 2) * invdet;
  r[0] = c0 * invdet;
  r[1] = c1 * invdet;
  r[2] = c2 * invdet;
  out = r;
}

int homography_from_matrix(const Mat3& m, Mat3& out) {
  Mat3 h = m;
  if (std::abs(h[8]) > 1e-12) {
    const double s = h[8];
    for (double& x : h) x /= s;
  }
  if (std::abs(det3(h)) <= 1e-12) return STITCH_B200_SingularHomography;
  out = h;
  return STITCH_B200_OK;
}

int homography_inverse(const Mat3& h, Mat3& out) {
  Mat3 inv;
  inverse3(h, inv);
  return homography_from_matrix(inv, out);
}

void homography_apply(const Mat3& h, double x, double y, double& ox, double& oy) {
  const double q0 = (h[0] * x + h[1] * y) + h[2] * 1.0;
  const double q1 = (h[3] * x + h[4] * y) + h[5] * 1.0;
  const double q2 = (h[6] * x + h[7] * y) + h[8] * 1.0;
  ox = q0 / q2;
  oy = q1 / q2;
}

// check_rotation (geometry.cpp:8-14)
static int check_rotation(const double* r) {
  Mat3 rm, rt, rrt;
  for (int i = 0; i < 9; ++i) rm[i] = r[i];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) rt[i * 3 + j] = r[j * 3 + i];
  mul3(rm, rt, rrt);
  double s = 0.0;
  for (int i = 0; i < 9; ++i) {
    const double d = rrt[i] - ((i % 4 == 0) ? 1.0 : 0.0);
    s += d * d;
  }
  if (std::sqrt(s) >= 1e-6 || det3(rm) < 0.0) return STITCH_B200_ConfigError;
  return STITCH_B200_OK;
}

int planar_homography(const stitch_b200_camera& c, Mat3& out) {
  int e = check_rotation(c.rotation);
  if (e != STITCH_B200_OK) return e;
  const Mat3 k = {c.fx, 0, c.cx, 0, c.fy, c.cy, 0, 0, 1};
  Mat3 cols;
  for (int i = 0; i < 3; ++i) {
    cols[i * 3 + 0] = c.rotation[i * 3 + 0];
    cols[i * 3 + 1] = c.rotation[i * 3 + 1];
    cols[i * 3 + 2] = c.translation[i];
  }
  Mat3 h;
  mul3(k, cols, h);
  if (std::abs(det3(h)) <= 1e-12) return STITCH_B200_DegeneratePose;
  return homography_from_matrix(h, out);
}

int pairwise_homography(const Mat3& hi, const Mat3& hj, Mat3& out) {
  Mat3 inv, p;
  inverse3(hj, inv);
  mul3(hi, inv, p);
  return homography_from_matrix(p, out);
}

Canvas compute_canvas(const std::vector<Mat3>& maps,
                      const std::vector<std::pair<int, int>>& sizes) {
  double min_x = std::numeric_limits<double>::max();
  double min_y = std::numeric_limits<double>::max();
  double max_x = std::numeric_limits<double>::lowest();
  double max_y = std::numeric_limits<double>::lowest();
  for (size_t v = 0; v < maps.size(); ++v) {
    const double w = sizes[v].first - 1.0, h = sizes[v].second - 1.0;
    const double cx[4] = {0.0, w, 0.0, w}, cy[4] = {0.0, 0.0, h, h};
    for (int k = 0; k < 4; ++k) {
      double X, Y;
      homography_apply(maps[v], cx[k], cy[k], X, Y);
      min_x = std::min(min_x, X);
      min_y = std::min(min_y, Y);
      max_x = std::max(max_x, X);
      max_y = std::max(max_y, Y);
    }
  }
  Canvas c;
  c.offx = std::floor(min_x);
  c.offy = std::floor(min_y);
  c.width = static_cast<int>(std::ceil(max_x) - c.offx) + 1;
  c.height = static_cast<int>(std::ceil(max_y) - c.offy) + 1;
  return c;
}

std::vector<PairSpec> build_pairs(int n_views, int reference, int topology) {
  std::vector<PairSpec> pairs;
  if (topology == 3) {
    // ring: k = (v - ref) mod N; distance min(k, N - k); partner one step
    // toward the reference (the k = N/2 view pairs with k - 1)
    for (int d = 1; d <= n_views / 2; ++d)
      for (int v = 0; v < n_views; ++v) {
        const int k = ((v - reference) % n_views + n_views) % n_views;
        if (std::min(k, n_views - k) != d) continue;
        const int partner = (k <= n_views / 2) ? (v - 1 + n_views) % n_views : (v + 1) % n_views;
        pairs.push_back({v, partner});
      }
    return pairs;
  }
  const int topo = (topology == 1 || topology == 2) ? topology : (n_views <= 3 ? 1 : 2);
  if (topo == 1) {
    for (int v = 0; v < n_views; ++v)
      if (v != reference) pairs.push_back({v, reference});
    return pairs;
  }
  for (int d = 1; d < n_views; ++d)
    for (int v = 0; v < n_views; ++v)
      if (std::abs(v - reference) == d)
        pairs.push_back({v, v < reference ? v + 1 : v - 1});
  return pairs;
}

static void rot_of(const stitch_b200_camera& c, Mat3& r) {
  for (int i = 0; i < 9; ++i) r[i] = c.rotation[i];
}

void cylinder_maps(const stitch_b200_config& cfg, std::vector<Mat3>& maps) {
  Mat3 rref, rrefT;
  rot_of(cfg.cams[cfg.reference], rref);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) rrefT[i * 3 + j] = rref[j * 3 + i];
  maps.resize(cfg.n_views);
  for (int v = 0; v < cfg.n_views; ++v) {
    const stitch_b200_camera& c = cfg.cams[v];
    const Mat3 k = {c.fx, 0, c.cx, 0, c.fy, c.cy, 0, 0, 1};
    Mat3 r, kr;
    rot_of(c, r);
    mul3(k, r, kr);
    mul3(kr, rrefT, maps[v]);
  }
}

Canvas cylinder_canvas(const stitch_b200_config& cfg, double f) {
  Mat3 rref;
  rot_of(cfg.cams[cfg.reference], rref);
  double hmin = std::numeric_limits<double>::max(), hmax = std::numeric_limits<double>::lowest();
  for (int v = 0; v < cfg.n_views; ++v) {
    const stitch_b200_camera& c = cfg.cams[v];
    Mat3 r, rT, m;
    rot_of(c, r);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) rT[i * 3 + j] = r[j * 3 + i];
    mul3(rref, rT, m);  // camera v -> reference frame
    const int W = cfg.width[v], H = cfg.height[v];
    auto visit = [&](double px, double py) {
      const double cx = (px - c.cx) / c.fx, cy = (py - c.cy) / c.fy;
      const double rx = (m[0] * cx + m[1] * cy) + m[2];
      const double ry = (m[3] * cx + m[4] * cy) + m[5];
      const double rz = (m[6] * cx + m[7] * cy) + m[8];
      const double h = ry / std::sqrt(rx * rx + rz * rz);
      hmin = std::min(hmin, h);
      hmax = std::max(hmax, h);
    };
    for (int x = 0; x < W; ++x) {
      visit(x, 0.0);
      visit(x, H - 1.0);
    }
    for (int y = 0; y < H; ++y) {
      visit(0.0, y);
      visit(W - 1.0, y);
    }
  }
  Canvas cv;
  cv.width = static_cast<int>(std::ceil(2.0 * M_PI * f));
  cv.offx = -std::floor(cv.width / 2.0);
  cv.offy = std::floor(hmin * f);
  cv.height = static_cast<int>(std::ceil(hmax * f) - cv.offy) + 1;
  return cv;
}

void lift_tables(const Canvas& c, double f, std::vector<double>& lsin, std::vector<double>& lcos,
                 std::vector<double>& lh) {
  lsin.resize(c.width);
  lcos.resize(c.width);
  lh.resize(c.height);
  for (int x = 0; x < c.width; ++x) {
    const double t = (x + c.offx) / f;
    lsin[x] = std::sin(t);
    lcos[x] = std::cos(t);
  }
  for (int y = 0; y < c.height; ++y) lh[y] = (y + c.offy) / f;
}

// ---------------------------------------------------------------------------
// feature refinement, host part
// ---------------------------------------------------------------------------
static int count_inliers(const std::vector<MatchPt>& m, const ScaleShift& p, double inlier_px,
                         std::vector<int>* idx, double* sse) {
  int count = 0;
  if (sse) *sse = 0.0;
  for (size_t i = 0; i < m.size(); ++i) {
    const double ex = p.s_x * m[i].ax + p.t_x - m[i].bx;
    const double ey = p.s_y * m[i].ay + p.t_y - m[i].by;
    const double e2 = ex * ex + ey * ey;
    if (e2 <= inlier_px * inlier_px) {
      ++count;
      if (idx) idx->push_back(static_cast<int>(i));
      if (sse) *sse += e2;
    }
  }
  return count;
}

// 1-D least squares b = s a + t over the inliers (features.cpp:260-278)
static bool fit_axis(const std::vector<MatchPt>& m, const std::vector<int>& idx, bool x_axis,
                     double& s, double& t) {
  double sa = 0, sb = 0, saa = 0, sab = 0;
  const double n = static_cast<double>(idx.size());
  for (int i : idx) {
    const double a = x_axis ? m[i].ax : m[i].ay;
    const double b = x_axis ? m[i].bx : m[i].by;
    sa += a;
    sb += b;
    saa += a * a;
    sab += a * b;
  }
  const double det = n * saa - sa * sa;
  if (std::abs(det) < 1e-9) return false;
  s = (n * sab - sa * sb) / det;
  t = (sb * saa - sa * sab) / det;
  return true;
}

int ransac_scale_translation(std::vector<MatchPt> m, int iterations, double inlier_px,
                             double min_scale, double max_scale, std::uint64_t seed,
                             ScaleShift& out) {
  if (m.size() < 2) return STITCH_B200_InsufficientMatches;
  // canonical order: the fit depends on the set and the seed only
  std::sort(m.begin(), m.end(), [](const MatchPt& a, const MatchPt& b) {
    return std::tie(a.ax, a.ay, a.bx, a.by, a.distance) <
           std::tie(b.ax, b.ay, b.bx, b.by, b.distance);
  });
  std::mt19937_64 rng(seed);
  std::uniform_int_distribution<std::size_t> pick(0, m.size() - 1);
  ScaleShift best;
  int best_count = -1;
  double best_sse = std::numeric_limits<double>::max();
  for (int it = 0; it < iterations; ++it) {
    const std::size_t i = pick(rng);
    const std::size_t j = pick(rng);
    if (i == j) continue;
    const double dax = m[j].ax - m[i].ax;
    const double day = m[j].ay - m[i].ay;
    if (std::abs(dax) < 1e-9 || std::abs(day) < 1e-9) continue;
    ScaleShift p;
    p.s_x = (m[j].bx - m[i].bx) / dax;
    p.s_y = (m[j].by - m[i].by) / day;
    p.t_x = m[i].bx - p.s_x * m[i].ax;
    p.t_y = m[i].by - p.s_y * m[i].ay;
    if (p.s_x < min_scale || p.s_x > max_scale || p.s_y < min_scale || p.s_y > max_scale) continue;
    double sse = 0.0;
    const int count = count_inliers(m, p, inlier_px, nullptr, &sse);
    if (count > best_count || (count == best_count && sse < best_sse)) {
      best = p;
      best_count = count;
      best_sse = sse;
    }
  }
  std::vector<int> inl;
  if (best_count > 0) count_inliers(m, best, inlier_px, &inl, nullptr);
  if (!(best_count >= 0 && (inl.size() * 2 >= m.size() || inl.size() >= 8)))
    return STITCH_B200_NoConsensus;
  ScaleShift refit = best;
  double s, t;
  if (fit_axis(m, inl, true, s, t)) {
    refit.s_x = s;
    refit.t_x = t;
  }
  if (fit_axis(m, inl, false, s, t)) {
    refit.s_y = s;
    refit.t_y = t;
  }
  out = refit;
  return STITCH_B200_OK;
}

void broaden(const int r[4], double margin, const int b[4], int out[4]) {
  const int mx = static_cast<int>(std::lround(margin * (r[2] - r[0])));
  const int my = static_cast<int>(std::lround(margin * (r[3] - r[1])));
  out[0] = std::max(b[0], r[0] - mx);
  out[1] = std::max(b[1], r[1] - my);
  out[2] = std::min(b[2], r[2] + mx);
  out[3] = std::min(b[3], r[3] + my);
}

}  // namespace stitch_b200_host
