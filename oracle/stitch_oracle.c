/*
 * stitch_oracle.c -- CPU ORACLE (test infrastructure only; see header).
 *
 * Restates the reference's per-frame path function by function.  Every
 * function cites the reference file:line it follows (paths relative to
 * /root/reference/proj).  Floating-point expressions keep the reference's
 * evaluation order; build with -O2 -ffp-contract=off (no FMA contraction),
 * which is also what the reference's default x86-64 build does.
 */
#include "stitch_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define SO_FAR_AWAY 1e9f /* flow.cpp:14 kFarAway */

static inline int imin(int a, int b) { return a < b ? a : b; }
static inline int imax(int a, int b) { return a > b ? a : b; }

static double now_seconds(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ------------------------------------------------------------------------ */
/* Frame helpers: frame.hpp:17-57                                            */
/* ------------------------------------------------------------------------ */

static int frame_alloc(so_frame* f, int w, int h, int with_mask,
                       uint8_t mask_fill) {
  f->width = w;
  f->height = h;
  f->data = (uint8_t*)calloc((size_t)w * h * 3 + 1, 1);
  f->mask = NULL;
  if (with_mask) {
    f->mask = (uint8_t*)malloc((size_t)w * h + 1);
    memset(f->mask, mask_fill, (size_t)w * h);
  }
  return f->data != NULL;
}

void so_free_frame(so_frame* f) {
  if (!f) return;
  free(f->data);
  free(f->mask);
  f->data = NULL;
  f->mask = NULL;
  f->width = f->height = 0;
}

static void frame_copy(so_frame* dst, const so_frame* src) {
  frame_alloc(dst, src->width, src->height, src->mask != NULL, 0);
  memcpy(dst->data, src->data, (size_t)src->width * src->height * 3);
  if (src->mask) memcpy(dst->mask, src->mask, (size_t)src->width * src->height);
}

/* Frame::valid_at, frame.hpp:44-47 */
static inline int valid_at(const so_frame* f, int x, int y) {
  if (x < 0 || y < 0 || x >= f->width || y >= f->height) return 0;
  return f->mask == NULL || f->mask[(size_t)y * f->width + x] != 0;
}

static inline const uint8_t* px(const so_frame* f, int x, int y) {
  return f->data + ((size_t)y * f->width + x) * 3;
}

/* quantize_channel, frame.cpp:30-35: round half away from zero, clamp. */
uint8_t so_quantize_channel(double v) {
  double r = round(v);
  if (r < 0.0) return 0;
  if (r > 255.0) return 255;
  return (uint8_t)r;
}

/* luma601 + to_luma, frame.hpp:63-65, frame.cpp:37-50 */
static inline float luma601(uint8_t r, uint8_t g, uint8_t b) {
  return 0.299f * (float)r + 0.587f * (float)g + 0.114f * (float)b;
}

static void to_luma(const so_frame* f, float* plane) {
  for (int y = 0; y < f->height; ++y) {
    for (int x = 0; x < f->width; ++x) {
      if (!valid_at(f, x, y)) {
        plane[(size_t)y * f->width + x] = 0.0f;
        continue;
      }
      const uint8_t* p = px(f, x, y);
      plane[(size_t)y * f->width + x] = luma601(p[0], p[1], p[2]);
    }
  }
}

/* check_region, frame.cpp:52-59 */
static int check_region(const so_frame* f, so_region r) {
  if (r.x1 <= r.x0 || r.y1 <= r.y0) return SO_EmptyRegion;
  if (r.x0 < 0 || r.y0 < 0 || r.x1 > f->width || r.y1 > f->height)
    return SO_EmptyRegion;
  return SO_OK;
}

/* crop_frame, frame.cpp:61-77 (output always carries a mask) */
static int crop_frame(const so_frame* f, so_region r, so_frame* out) {
  int e = check_region(f, r);
  if (e != SO_OK) return e;
  const int w = r.x1 - r.x0, h = r.y1 - r.y0;
  frame_alloc(out, w, h, 1, 0);
  for (int y = 0; y < h; ++y) {
    for (int x = 0; x < w; ++x) {
      const int sx = r.x0 + x, sy = r.y0 + y;
      const uint8_t* s = px(f, sx, sy);
      uint8_t* d = out->data + ((size_t)y * w + x) * 3;
      d[0] = s[0];
      d[1] = s[1];
      d[2] = s[2];
      out->mask[(size_t)y * w + x] = valid_at(f, sx, sy) ? 1 : 0;
    }
  }
  return SO_OK;
}

/* sample_bilinear, frame.cpp:79-109.  j (rows) outer, i (cols) inner;
 * zero/negative weights and invalid neighbours drop out; double
 * accumulation, renormalised, cast to float. */
int so_sample_bilinear(const so_frame* f, double x, double y, float rgb[3]) {
  const double fx0 = floor(x);
  const double fy0 = floor(y);
  const int x0 = (int)fx0;
  const int y0 = (int)fy0;
  const double ax = x - fx0;
  const double ay = y - fy0;
  const int xs[2] = {x0, x0 + 1};
  const int ys[2] = {y0, y0 + 1};
  const double wx[2] = {1.0 - ax, ax};
  const double wy[2] = {1.0 - ay, ay};
  double wsum = 0.0;
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
  for (int j = 0; j < 2; ++j) {
    for (int i = 0; i < 2; ++i) {
      const double w = wx[i] * wy[j];
      if (w <= 0.0) continue;
      if (!valid_at(f, xs[i], ys[j])) continue;
      const uint8_t* p = px(f, xs[i], ys[j]);
      acc0 += w * (double)p[0];
      acc1 += w * (double)p[1];
      acc2 += w * (double)p[2];
      wsum += w;
    }
  }
  if (wsum <= 0.0) return 0;
  rgb[0] = (float)(acc0 / wsum);
  rgb[1] = (float)(acc1 / wsum);
  rgb[2] = (float)(acc2 / wsum);
  return 1;
}

/* ------------------------------------------------------------------------ */
/* Histogram: histogram.hpp:12-22, histogram.cpp:5-33                        */
/* ------------------------------------------------------------------------ */

int so_compute_histogram(const so_frame* f, so_region r, so_hist* out) {
  memset(out, 0, sizeof(*out));
  int e = check_region(f, r);
  if (e != SO_OK) return e;
  for (int y = r.y0; y < r.y1; ++y) {
    for (int x = r.x0; x < r.x1; ++x) {
      if (!valid_at(f, x, y)) continue;
      const uint8_t* p = px(f, x, y);
      ++out->bins[0][p[0]];
      ++out->bins[1][p[1]];
      ++out->bins[2][p[2]];
      ++out->total;
    }
  }
  if (out->total == 0) return SO_EmptyRegion;
  return SO_OK;
}

int so_cdf(const so_hist* h, double out[3][256]) {
  if (h->total == 0) return SO_EmptyHistogram;
  for (int c = 0; c < 3; ++c) {
    uint64_t run = 0;
    for (int v = 0; v < 256; ++v) {
      run += h->bins[c][v];
      out[c][v] = (double)run / (double)h->total;
    }
  }
  return SO_OK;
}

/* ------------------------------------------------------------------------ */
/* 3x3 linear algebra at the Eigen boundary (PARITY UNPINNED at last ulp).   */
/* ------------------------------------------------------------------------ */

/* Eigen's 3x3 cofactor inverse (Eigen/src/LU/InverseImpl.h,
 * compute_inverse<...,3>): cofactors of column 0, det = sum(cof .* col0),
 * inv(i,j) = cofactor(j,i) * (1/det).  Used at pipeline.cpp:40 and
 * geometry.cpp:30,54,60. */
static inline double cof3(const double* m, int i, int j) {
  const int i1 = (i + 1) % 3, i2 = (i + 2) % 3;
  const int j1 = (j + 1) % 3, j2 = (j + 2) % 3;
  return m[i1 * 3 + j1] * m[i2 * 3 + j2] - m[i1 * 3 + j2] * m[i2 * 3 + j1];
}

void so_inverse3(const double m[9], double out[9]) {
  const double c0 = cof3(m, 0, 0), c1 = cof3(m, 1, 0), c2 = cof3(m, 2, 0);
  const double det = (c0 * m[0] + c1 * m[3]) + c2 * m[6];
  const double invdet = 1.0 / det;
  double r[9];
  r[1 * 3 + 0] = cof3(m, 0, 1) * invdet;
  r[1 * 3 + 1] = cof3(m, 1, 1) * invdet;
  r[2 * 3 + 0] = cof3(m, 0, 2) * invdet;
  r[1 * 3 + 2] = cof3(m, 2, 1) * invdet;
  r[2 * 3 + 1] = cof3(m, 1, 2) * invdet;
  r[2 * 3 + 2] = cof3(m, 2, 2) * invdet;
  r[0] = c0 * invdet;
  r[1] = c1 * invdet;
  r[2] = c2 * invdet;
  memcpy(out, r, sizeof(r));
}

double so_det3(const double m[9]) {
  const double c0 = cof3(m, 0, 0), c1 = cof3(m, 1, 0), c2 = cof3(m, 2, 0);
  return (c0 * m[0] + c1 * m[3]) + c2 * m[6];
}

static void mul3(const double* a, const double* b, double* out) {
  double r[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r[i * 3 + j] = (a[i * 3 + 0] * b[0 * 3 + j] + a[i * 3 + 1] * b[1 * 3 + j]) +
                     a[i * 3 + 2] * b[2 * 3 + j];
  memcpy(out, r, sizeof(r));
}

/* Homography::from_matrix, geometry.cpp:16-26 */
static int homography_from_matrix(const double* m, double* out) {
  double h[9];
  memcpy(h, m, sizeof(h));
  if (fabs(h[8]) > 1e-12) {
    const double s = h[8];
    for (int i = 0; i < 9; ++i) h[i] /= s;
  }
  if (fabs(so_det3(h)) <= 1e-12) return SO_SingularHomography;
  memcpy(out, h, sizeof(h));
  return SO_OK;
}

/* Homography::apply, geometry.cpp:33-36 */
static void homography_apply(const double* h, double x, double y, double* ox,
                             double* oy) {
  const double q0 = (h[0] * x + h[1] * y) + h[2] * 1.0;
  const double q1 = (h[3] * x + h[4] * y) + h[5] * 1.0;
  const double q2 = (h[6] * x + h[7] * y) + h[8] * 1.0;
  *ox = q0 / q2;
  *oy = q1 / q2;
}

/* check_rotation, geometry.cpp:8-14 */
static int check_rotation(const double* r) {
  double rrt[9];
  double rt[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) rt[i * 3 + j] = r[j * 3 + i];
  mul3(r, rt, rrt);
  double s = 0.0;
  for (int i = 0; i < 9; ++i) {
    const double d = rrt[i] - ((i % 4 == 0) ? 1.0 : 0.0);
    s += d * d;
  }
  if (sqrt(s) >= 1e-6 || so_det3(r) < 0.0) return SO_ConfigError;
  return SO_OK;
}

/* planar_homography, geometry.cpp:38-51: K * [r1 r2 t], normalised. */
static int planar_homography(const so_camera* c, double* out) {
  int e = check_rotation(c->rotation);
  if (e != SO_OK) return e;
  const double k[9] = {c->fx, 0, c->cx, 0, c->fy, c->cy, 0, 0, 1};
  double cols[9];
  for (int i = 0; i < 3; ++i) {
    cols[i * 3 + 0] = c->rotation[i * 3 + 0];
    cols[i * 3 + 1] = c->rotation[i * 3 + 1];
    cols[i * 3 + 2] = c->translation[i];
  }
  double h[9];
  mul3(k, cols, h);
  if (fabs(so_det3(h)) <= 1e-12) return SO_DegeneratePose;
  return homography_from_matrix(h, out);
}

/* pairwise_homography, geometry.cpp:53-56: normalised h_i * h_j^-1 */
static int pairwise_homography(const double* hi, const double* hj,
                               double* out) {
  double inv[9], p[9];
  so_inverse3(hj, inv);
  mul3(hi, inv, p);
  return homography_from_matrix(p, out);
}

/* ------------------------------------------------------------------------ */
/* Warp: warp_frame_parallel, pipeline.cpp:38-66 (== geometry.cpp:58-83)     */
/* ------------------------------------------------------------------------ */

int so_warp_frame(const so_frame* src, const double inv[9], int cw, int ch,
                  double offx, double offy, int threads, so_frame* out) {
  frame_alloc(out, cw, ch, 1, 0);
  int any = 0;
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1) reduction(| : any)
  for (int y = 0; y < ch; ++y) {
    for (int x = 0; x < cw; ++x) {
      const double X = (double)x + offx;
      const double Y = (double)y + offy;
      const double sx0 = (inv[0] * X + inv[1] * Y) + inv[2] * 1.0;
      const double sy0 = (inv[3] * X + inv[4] * Y) + inv[5] * 1.0;
      const double sz0 = (inv[6] * X + inv[7] * Y) + inv[8] * 1.0;
      if (fabs(sz0) < 1e-12) continue;
      float rgb[3];
      if (!so_sample_bilinear(src, sx0 / sz0, sy0 / sz0, rgb)) continue;
      uint8_t* p = out->data + ((size_t)y * cw + x) * 3;
      p[0] = so_quantize_channel(rgb[0]);
      p[1] = so_quantize_channel(rgb[1]);
      p[2] = so_quantize_channel(rgb[2]);
      out->mask[(size_t)y * cw + x] = 1;
      any = 1;
    }
  }
  if (!any) return SO_EmptyProjection;
  return SO_OK;
}

/* Warp over a lifted canvas (extension).  lsin == NULL: the reference's
 * planar lift (x + offx, y + offy, 1), identical arithmetic to
 * so_warp_frame since a*1.0 == a; otherwise the cylindrical lift
 * (sin t[x], h[y], cos t[x]) and points behind the camera are invalid. */
int so_warp_frame_lift(const so_frame* src, const double a[9], int cw, int ch,
                       double offx, double offy, const double* lsin,
                       const double* lcos, const double* lh, int threads,
                       so_frame* out) {
  if (!lsin) return so_warp_frame(src, a, cw, ch, offx, offy, threads, out);
  frame_alloc(out, cw, ch, 1, 0);
  int any = 0;
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1) reduction(| : any)
  for (int y = 0; y < ch; ++y) {
    for (int x = 0; x < cw; ++x) {
      const double L0 = lsin[x], L1 = lh[y], L2 = lcos[x];
      const double sx0 = (a[0] * L0 + a[1] * L1) + a[2] * L2;
      const double sy0 = (a[3] * L0 + a[4] * L1) + a[5] * L2;
      const double sz0 = (a[6] * L0 + a[7] * L1) + a[8] * L2;
      if (fabs(sz0) < 1e-12) continue;
      if (!(sz0 > 0.0)) continue;
      float rgb[3];
      if (!so_sample_bilinear(src, sx0 / sz0, sy0 / sz0, rgb)) continue;
      uint8_t* p = out->data + ((size_t)y * cw + x) * 3;
      p[0] = so_quantize_channel(rgb[0]);
      p[1] = so_quantize_channel(rgb[1]);
      p[2] = so_quantize_channel(rgb[2]);
      out->mask[(size_t)y * cw + x] = 1;
      any = 1;
    }
  }
  if (!any) return SO_EmptyProjection;
  return SO_OK;
}

/* overlap_regions, geometry.cpp:85-117 (bounds only) */
static int overlap_bounds(const so_frame* a, const so_frame* b, so_region* r) {
  if (a->width != b->width || a->height != b->height) return SO_ShapeMismatch;
  int x0 = a->width, y0 = a->height, x1 = 0, y1 = 0;
  for (int y = 0; y < a->height; ++y) {
    for (int x = 0; x < a->width; ++x) {
      if (valid_at(a, x, y) && valid_at(b, x, y)) {
        x0 = imin(x0, x);
        y0 = imin(y0, y);
        x1 = imax(x1, x + 1);
        y1 = imax(y1, y + 1);
      }
    }
  }
  if (x1 <= x0 || y1 <= y0) return SO_NoOverlap;
  r->x0 = x0;
  r->y0 = y0;
  r->x1 = x1;
  r->y1 = y1;
  return SO_OK;
}

static void mask_bbox(const so_frame* a, so_region* r) {
  int x0 = a->width, y0 = a->height, x1 = 0, y1 = 0;
  for (int y = 0; y < a->height; ++y)
    for (int x = 0; x < a->width; ++x)
      if (valid_at(a, x, y)) {
        x0 = imin(x0, x);
        y0 = imin(y0, y);
        x1 = imax(x1, x + 1);
        y1 = imax(y1, y + 1);
      }
  r->x0 = x0;
  r->y0 = y0;
  r->x1 = x1;
  r->y1 = y1;
}

/* ------------------------------------------------------------------------ */
/* Color transfer (3D-M): color_transfer.cpp:28-191                          */
/* ------------------------------------------------------------------------ */

/* histogram_specification, color_transfer.cpp:28-55 */
int so_histogram_specification(const so_hist* src, const so_hist* ref,
                               uint8_t lut[3][256]) {
  if (src->total == 0 || ref->total == 0) return SO_EmptyHistogram;
  for (int c = 0; c < 3; ++c) {
    uint64_t cum_ref[256];
    uint64_t run = 0;
    for (int v = 0; v < 256; ++v) {
      run += ref->bins[c][v];
      cum_ref[v] = run;
    }
    uint64_t cum_src = 0;
    int u = 0;
    for (int v = 0; v < 256; ++v) {
      cum_src += src->bins[c][v];
      while (u < 255 && cum_ref[u] * src->total < cum_src * ref->total) ++u;
      lut[c][v] = (uint8_t)u;
    }
  }
  return SO_OK;
}

/* Symmetric 3x3 eigenvalues by cyclic Jacobi rotations; for the PSD normal
 * matrix these are its singular values (JacobiSVD at
 * color_transfer.cpp:88-89).  Sorted descending by magnitude. */
void so_sym3_eigen(const double a_in[9], double ev[3]) {
  double a[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) a[i][j] = a_in[i * 3 + j];
  for (int sweep = 0; sweep < 32; ++sweep) {
    const double off = (fabs(a[0][1]) + fabs(a[0][2])) + fabs(a[1][2]);
    if (off == 0.0) break;
    for (int p = 0; p < 2; ++p) {
      for (int q = p + 1; q < 3; ++q) {
        const double apq = a[p][q];
        if (apq == 0.0) continue;
        const double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) /
                         (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0);
        const double s = t * c;
        for (int k = 0; k < 3; ++k) {
          const double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - s * akq;
          a[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          const double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - s * aqk;
          a[q][k] = s * apk + c * aqk;
        }
        a[p][q] = 0.0;
        a[q][p] = 0.0;
      }
    }
  }
  double e[3] = {fabs(a[0][0]), fabs(a[1][1]), fabs(a[2][2])};
  for (int i = 0; i < 3; ++i)
    for (int j = i + 1; j < 3; ++j)
      if (e[j] > e[i]) {
        const double t = e[i];
        e[i] = e[j];
        e[j] = t;
      }
  ev[0] = e[0];
  ev[1] = e[1];
  ev[2] = e[2];
}

/* Eigen LDLT<Matrix3d, Lower> with diagonal pivoting
 * (Eigen/src/Cholesky/LDLT.h, ldlt_inplace<Lower>::unblocked and
 * LDLT::_solve_impl), as used at color_transfer.cpp:96. */
void so_ldlt_solve3(const double a_in[9], const double b_in[9], double x[9]) {
  double m[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m[i][j] = a_in[i * 3 + j];
  int tr[3];
  double temp[3];
  const int n = 3;
  for (int k = 0; k < n; ++k) {
    int big = k;
    double bigv = fabs(m[k][k]);
    for (int i = k + 1; i < n; ++i)
      if (fabs(m[i][i]) > bigv) {
        bigv = fabs(m[i][i]);
        big = i;
      }
    tr[k] = big;
    if (k != big) {
      for (int j = 0; j < k; ++j) {
        const double t = m[k][j];
        m[k][j] = m[big][j];
        m[big][j] = t;
      }
      for (int i = big + 1; i < n; ++i) {
        const double t = m[i][k];
        m[i][k] = m[i][big];
        m[i][big] = t;
      }
      {
        const double t = m[k][k];
        m[k][k] = m[big][big];
        m[big][big] = t;
      }
      for (int i = k + 1; i < big; ++i) {
        const double t = m[i][k];
        m[i][k] = m[big][i];
        m[big][i] = t;
      }
    }
    const int rs = n - k - 1;
    if (k > 0) {
      for (int j = 0; j < k; ++j) temp[j] = m[j][j] * m[k][j];
      double dot = 0.0;
      for (int j = 0; j < k; ++j) dot = (j == 0) ? m[k][j] * temp[j] : dot + m[k][j] * temp[j];
      m[k][k] -= dot;
      for (int i = k + 1; i < n; ++i) {
        double d = 0.0;
        for (int j = 0; j < k; ++j) d = (j == 0) ? m[i][j] * temp[j] : d + m[i][j] * temp[j];
        m[i][k] -= d;
      }
    }
    const double akk = m[k][k];
    const int valid = fabs(akk) > 0.0;
    if (k == 0 && !valid) {
      for (int j = 0; j < n; ++j) {
        tr[j] = j;
        for (int i = j + 1; i < n; ++i) m[i][j] = 0.0;
      }
      break;
    }
    if (rs > 0 && valid)
      for (int i = k + 1; i < n; ++i) m[i][k] /= akk;
  }
  /* solve for each of the 3 right-hand-side columns */
  for (int col = 0; col < 3; ++col) {
    double d[3] = {b_in[0 * 3 + col], b_in[1 * 3 + col], b_in[2 * 3 + col]};
    for (int k = 0; k < n; ++k) {
      const double t = d[k];
      d[k] = d[tr[k]];
      d[tr[k]] = t;
    }
    for (int i = 1; i < n; ++i)
      for (int j = 0; j < i; ++j) d[i] -= m[i][j] * d[j];
    for (int i = 0; i < n; ++i) {
      if (fabs(m[i][i]) > DBL_MIN)
        d[i] /= m[i][i];
      else
        d[i] = 0.0;
    }
    /* L^T x = y: Eigen's triangular_solve_matrix (row-major U = L^T view)
     * accumulates b = sum_{j>i} U_ij x_j from 0 first, then x_i = (x_i - b)
     * -- pinned against the compiled reference (tests/test_ref_pin.py). */
    for (int i = n - 2; i >= 0; --i) {
      double b = 0.0;
      for (int j = i + 1; j < n; ++j) b += m[j][i] * d[j];
      d[i] = d[i] - b;
    }
    for (int k = n - 1; k >= 0; --k) {
      const double t = d[k];
      d[k] = d[tr[k]];
      d[tr[k]] = t;
    }
    for (int i = 0; i < 3; ++i) x[i * 3 + col] = d[i];
  }
}

/* solve_color_matrix tail, color_transfer.cpp:87-98, given the exact
 * moments normal = X^T X and xty = X^T Y of the stacked window rows. */
static int solve_from_moments(const double normal[9], const double xty[9],
                              long long n, double m[9], double* min_sv) {
  double sv[3];
  so_sym3_eigen(normal, sv);
  if (n < 3 || sv[2] < 1e-8 * sv[0]) return SO_RankDeficient;
  so_ldlt_solve3(normal, xty, m);
  if (min_sv) *min_sv = sv[2];
  return SO_OK;
}

/* solve_color_matrix, color_transfer.cpp:73-99 (rows stacked newest->oldest) */
int so_solve_color_matrix(int entries, const int* rows,
                          const double* const* src, const double* const* tgt,
                          double m[9], double* min_singular) {
  if (entries <= 0) return SO_MissingState;
  double normal[9] = {0}, xty[9] = {0};
  long long n = 0;
  for (int e = 0; e < entries; ++e) {
    for (int r = 0; r < rows[e]; ++r) {
      const double* xs = src[e] + (size_t)r * 3;
      const double* ys = tgt[e] + (size_t)r * 3;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
          normal[a * 3 + b] += xs[a] * xs[b];
          xty[a * 3 + b] += xs[a] * ys[b];
        }
    }
    n += rows[e];
  }
  return solve_from_moments(normal, xty, n, m, min_singular);
}

/* apply_matrix_rows, pipeline.cpp:68-82: rgb' = quantize(rgb * M) on the
 * valid pixels of the whole frame. */
void so_apply_color_matrix_rows(so_frame* f, const double m[9], int threads) {
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
  for (int y = 0; y < f->height; ++y) {
    for (int x = 0; x < f->width; ++x) {
      if (!valid_at(f, x, y)) continue;
      uint8_t* p = f->data + ((size_t)y * f->width + x) * 3;
      const double r = p[0], g = p[1], b = p[2];
      const double o0 = (r * m[0] + g * m[3]) + b * m[6];
      const double o1 = (r * m[1] + g * m[4]) + b * m[7];
      const double o2 = (r * m[2] + g * m[5]) + b * m[8];
      p[0] = so_quantize_channel(o0);
      p[1] = so_quantize_channel(o1);
      p[2] = so_quantize_channel(o2);
    }
  }
}

/* TransferWindow, color_transfer.hpp:40-61 / color_transfer.cpp:8-26.
 * Rows are u8 triples (the reference stores the same integer values as
 * doubles). Newest first. */
typedef struct {
  int rows;
  uint8_t* src; /* rows x 3 raw overlap pixels */
  uint8_t* tgt; /* rows x 3 specification-revised pixels */
} so_wentry;

typedef struct {
  int capacity;
  int size;
  so_wentry e[3];
} so_window;

static void window_push(so_window* w, so_wentry ne) {
  if (w->size == w->capacity) {
    free(w->e[w->size - 1].src);
    free(w->e[w->size - 1].tgt);
    w->size--;
  }
  for (int i = w->size; i > 0; --i) w->e[i] = w->e[i - 1];
  w->e[0] = ne;
  w->size++;
}

static void window_free(so_window* w) {
  for (int i = 0; i < w->size; ++i) {
    free(w->e[i].src);
    free(w->e[i].tgt);
  }
  w->size = 0;
}

/* transfer_step, color_transfer.cpp:133-191, as driven by process_frame
 * (pipeline.cpp:281-299).  The corrected-overlap copy of line 189 is
 * discarded by the caller and is not computed.  On EmptyRegion the window
 * is untouched; on RankDeficient it is still updated. */
static int transfer_step(const so_frame* source, const so_frame* reference,
                         so_region ov, so_window* window, double m[9],
                         int* rank_deficient) {
  int e = check_region(source, ov);
  if (e != SO_OK) return e;
  e = check_region(reference, ov);
  if (e != SO_OK) return e;
  so_hist hs, hr;
  memset(&hs, 0, sizeof(hs));
  memset(&hr, 0, sizeof(hr));
  const int w = ov.x1 - ov.x0, h = ov.y1 - ov.y0;
  uint8_t* raw = (uint8_t*)malloc((size_t)w * h * 3 + 1);
  int n = 0;
  for (int dy = 0; dy < h; ++dy) {
    for (int dx = 0; dx < w; ++dx) {
      const int x = ov.x0 + dx, y = ov.y0 + dy;
      if (!valid_at(source, x, y) || !valid_at(reference, x, y)) continue;
      const uint8_t* s = px(source, x, y);
      const uint8_t* r = px(reference, x, y);
      for (int c = 0; c < 3; ++c) {
        ++hs.bins[c][s[c]];
        ++hr.bins[c][r[c]];
      }
      ++hs.total;
      ++hr.total;
      raw[(size_t)n * 3 + 0] = s[0];
      raw[(size_t)n * 3 + 1] = s[1];
      raw[(size_t)n * 3 + 2] = s[2];
      ++n;
    }
  }
  if (n == 0) {
    free(raw);
    return SO_EmptyRegion;
  }
  uint8_t lut[3][256];
  so_histogram_specification(&hs, &hr, lut);
  uint8_t* rev = (uint8_t*)malloc((size_t)n * 3);
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < 3; ++c) rev[(size_t)i * 3 + c] = lut[c][raw[(size_t)i * 3 + c]];
  so_wentry ne = {n, raw, rev};
  window_push(window, ne);

  double normal[9] = {0}, xty[9] = {0};
  long long total = 0;
  for (int k = 0; k < window->size; ++k) {
    const so_wentry* en = &window->e[k];
    for (int r = 0; r < en->rows; ++r) {
      const uint8_t* xs = en->src + (size_t)r * 3;
      const uint8_t* ys = en->tgt + (size_t)r * 3;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
          normal[a * 3 + b] += (double)xs[a] * (double)xs[b];
          xty[a * 3 + b] += (double)xs[a] * (double)ys[b];
        }
    }
    total += en->rows;
  }
  *rank_deficient = 0;
  if (solve_from_moments(normal, xty, total, m, NULL) != SO_OK) {
    for (int i = 0; i < 9; ++i) m[i] = (i % 4 == 0) ? 1.0 : 0.0;
    *rank_deficient = 1;
  }
  return SO_OK;
}

/* ------------------------------------------------------------------------ */
/* Global balance: color_balance.cpp:8-104, pipeline.cpp:84-96,336-355        */
/* ------------------------------------------------------------------------ */

int so_find_thresholds(const so_hist* h, double lambda, int m1o[3],
                       int m2o[3]) {
  if (h->total == 0) return SO_EmptyHistogram;
  if (!(lambda > 0.0 && lambda < 0.5)) return SO_ConfigError;
  const double total = (double)h->total;
  for (int c = 0; c < 3; ++c) {
    uint64_t run = 0;
    int m1 = 255, m2 = 255, have1 = 0, have2 = 0;
    for (int v = 0; v < 256; ++v) {
      run += h->bins[c][v];
      const double cdf = (double)run / total;
      if (!have1 && cdf >= lambda) {
        m1 = v;
        have1 = 1;
      }
      if (!have2 && cdf >= 1.0 - lambda) {
        m2 = v;
        have2 = 1;
        break;
      }
    }
    m1o[c] = m1;
    m2o[c] = m2;
  }
  return SO_OK;
}

/* smooth_thresholds, color_balance.cpp:40-63: mean of the newest <= 3
 * entries (history newest last), lround, swap if crossed. */
void so_smooth_thresholds(int n_hist, const int (*m1)[3], const int (*m2)[3],
                          int out_m1[3], int out_m2[3]) {
  const int n = n_hist < 3 ? n_hist : 3;
  const int start = n_hist - n;
  for (int c = 0; c < 3; ++c) {
    double s1 = 0.0, s2 = 0.0;
    for (int i = start; i < n_hist; ++i) {
      s1 += m1[i][c];
      s2 += m2[i][c];
    }
    int a = (int)lround(s1 / (double)n);
    int b = (int)lround(s2 / (double)n);
    if (a > b) {
      const int t = a;
      a = b;
      b = t;
    }
    out_m1[c] = a;
    out_m2[c] = b;
  }
}

/* balance_curve_value, color_balance.cpp:65-86 */
double so_balance_curve_value(double x, int m1, int m2, double gamma_dark,
                              double gamma_bright, int tbi, int twi) {
  const double tb = tbi, tw = twi;
  if (m1 >= m2) return tb + (tw - tb) * (x / 255.0);
  const double lm1 = tb + (tw - tb) * ((double)m1 / 255.0);
  const double lm2 = tb + (tw - tb) * ((double)m2 / 255.0);
  if (x <= m1) {
    if (m1 == 0) return tb;
    return tb + (lm1 - tb) * pow(x / m1, gamma_dark);
  }
  if (x >= m2) {
    if (m2 == 255) return tw;
    return lm2 + (tw - lm2) * pow((x - m2) / (255.0 - m2), gamma_bright);
  }
  return lm1 + (lm2 - lm1) * (x - m1) / (m2 - m1);
}

/* build_curve, color_balance.cpp:88-104 */
int so_build_curve(const int m1[3], const int m2[3], double gamma_dark,
                   double gamma_bright, int tb, int tw, uint8_t lut[3][256]) {
  if (!(gamma_dark > 0.0 && gamma_bright > 0.0)) return SO_ConfigError;
  if (tb > tw) return SO_ConfigError;
  for (int c = 0; c < 3; ++c)
    for (int v = 0; v < 256; ++v)
      lut[c][v] = so_quantize_channel(so_balance_curve_value(
          (double)v, m1[c], m2[c], gamma_dark, gamma_bright, tb, tw));
  return SO_OK;
}

/* ------------------------------------------------------------------------ */
/* Dense flow: flow.cpp:16-187                                               */
/* ------------------------------------------------------------------------ */

typedef struct {
  int w, h;
  float* p;
} plane;

static plane plane_new(int w, int h) {
  plane r = {w, h, (float*)calloc((size_t)w * h + 1, sizeof(float))};
  return r;
}
#define PL(pl, y, x) ((pl).p[(size_t)(y) * (pl).w + (x)])

/* downsample_half, flow.cpp:16-31 */
static plane downsample_half(plane src) {
  const int w = imax(1, src.w / 2), h = imax(1, src.h / 2);
  plane out = plane_new(w, h);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const int x0 = 2 * x, y0 = 2 * y;
      const int x1 = imin(x0 + 1, src.w - 1), y1 = imin(y0 + 1, src.h - 1);
      PL(out, y, x) = 0.25f * (PL(src, y0, x0) + PL(src, y0, x1) +
                               PL(src, y1, x0) + PL(src, y1, x1));
    }
  return out;
}

/* resize_bilinear, flow.cpp:33-55 */
static plane resize_bilinear(plane src, int w, int h, float value_scale) {
  plane out = plane_new(w, h);
  const int sw = src.w, sh = src.h;
  const float fx = w > 1 ? (float)(sw - 1) / (float)(w - 1) : 0.0f;
  const float fy = h > 1 ? (float)(sh - 1) / (float)(h - 1) : 0.0f;
  for (int y = 0; y < h; ++y) {
    const float sy = (float)y * fy;
    const int y0 = imin(sh - 1, (int)sy);
    const int y1 = imin(sh - 1, y0 + 1);
    const float ay = sy - (float)y0;
    for (int x = 0; x < w; ++x) {
      const float sx = (float)x * fx;
      const int x0 = imin(sw - 1, (int)sx);
      const int x1 = imin(sw - 1, x0 + 1);
      const float ax = sx - (float)x0;
      const float top = (1.0f - ax) * PL(src, y0, x0) + ax * PL(src, y0, x1);
      const float bot = (1.0f - ax) * PL(src, y1, x0) + ax * PL(src, y1, x1);
      PL(out, y, x) = value_scale * ((1.0f - ay) * top + ay * bot);
    }
  }
  return out;
}

/* std::clamp(v, lo, hi) */
static inline float clampf_std(float v, float lo, float hi) {
  return (v < lo) ? lo : (hi < v) ? hi : v;
}

/* sample_clamped, flow.cpp:57-70 */
static inline float sample_clamped(plane img, float x, float y) {
  const int w = img.w, h = img.h;
  x = clampf_std(x, 0.0f, (float)(w - 1));
  y = clampf_std(y, 0.0f, (float)(h - 1));
  const int x0 = imin(w - 1, (int)x);
  const int y0 = imin(h - 1, (int)y);
  const int x1 = imin(w - 1, x0 + 1);
  const int y1 = imin(h - 1, y0 + 1);
  const float ax = x - (float)x0;
  const float ay = y - (float)y0;
  return (1.0f - ay) * ((1.0f - ax) * PL(img, y0, x0) + ax * PL(img, y0, x1)) +
         ay * ((1.0f - ax) * PL(img, y1, x0) + ax * PL(img, y1, x1));
}

/* refine_level, flow.cpp:74-136 */
static void refine_level(plane a, plane b, plane* u, plane* v, int iterations,
                         double alpha, int threads) {
  const int w = a.w, h = a.h;
  const float alpha2 = (float)(alpha * alpha);
  const int warps = 5;
  const int sweeps = imax(1, iterations / warps);
  plane bw = plane_new(w, h), ix = plane_new(w, h), iy = plane_new(w, h),
        it = plane_new(w, h), u0 = plane_new(w, h), v0 = plane_new(w, h),
        un = plane_new(w, h), vn = plane_new(w, h);
  const int nt = threads > 0 ? threads : 1;
  for (int warp = 0; warp < warps; ++warp) {
    plane U = *u, V = *v;
#pragma omp parallel for schedule(static) num_threads(nt)
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x)
        PL(bw, y, x) = sample_clamped(b, (float)x + PL(U, y, x),
                                      (float)y + PL(V, y, x));
    memcpy(u0.p, U.p, sizeof(float) * (size_t)w * h);
    memcpy(v0.p, V.p, sizeof(float) * (size_t)w * h);
#pragma omp parallel for schedule(static) num_threads(nt)
    for (int y = 0; y < h; ++y) {
      const int ym = imax(0, y - 1), yp = imin(h - 1, y + 1);
      for (int x = 0; x < w; ++x) {
        const int xm = imax(0, x - 1), xp = imin(w - 1, x + 1);
        PL(ix, y, x) = 0.25f * (PL(a, y, xp) - PL(a, y, xm) + PL(bw, y, xp) -
                                PL(bw, y, xm));
        PL(iy, y, x) = 0.25f * (PL(a, yp, x) - PL(a, ym, x) + PL(bw, yp, x) -
                                PL(bw, ym, x));
        PL(it, y, x) = PL(bw, y, x) - PL(a, y, x);
      }
    }
    for (int sweep = 0; sweep < sweeps; ++sweep) {
      plane Uc = *u, Vc = *v;
#pragma omp parallel for schedule(static) num_threads(nt)
      for (int y = 0; y < h; ++y) {
        const int ym = imax(0, y - 1), yp = imin(h - 1, y + 1);
        for (int x = 0; x < w; ++x) {
          const int xm = imax(0, x - 1), xp = imin(w - 1, x + 1);
          const float ubar = 0.25f * (PL(Uc, y, xm) + PL(Uc, y, xp) +
                                      PL(Uc, ym, x) + PL(Uc, yp, x));
          const float vbar = 0.25f * (PL(Vc, y, xm) + PL(Vc, y, xp) +
                                      PL(Vc, ym, x) + PL(Vc, yp, x));
          const float gx = PL(ix, y, x);
          const float gy = PL(iy, y, x);
          const float c = PL(it, y, x) - gx * PL(u0, y, x) - gy * PL(v0, y, x);
          const float denom = alpha2 + gx * gx + gy * gy;
          const float common = (gx * ubar + gy * vbar + c) / denom;
          PL(un, y, x) = ubar - gx * common;
          PL(vn, y, x) = vbar - gy * common;
        }
      }
      plane t = *u;
      *u = un;
      un = t;
      t = *v;
      *v = vn;
      vn = t;
    }
  }
  free(bw.p);
  free(ix.p);
  free(iy.p);
  free(it.p);
  free(u0.p);
  free(v0.p);
  free(un.p);
  free(vn.p);
}

/* dense_flow, flow.cpp:140-187.  u, v: a.width*a.height floats. */
int so_dense_flow(const so_frame* ra, const so_frame* rb, int levels,
                  int iterations, double smoothness, int threads, float* uo,
                  float* vo) {
  if (ra->width != rb->width || ra->height != rb->height)
    return SO_ShapeMismatch;
  if (ra->width < 16 || ra->height < 16) return SO_TooSmall;
  plane pa[32], pb[32];
  int np = 1;
  pa[0] = plane_new(ra->width, ra->height);
  pb[0] = plane_new(rb->width, rb->height);
  to_luma(ra, pa[0].p);
  to_luma(rb, pb[0].p);
  for (int l = 1; l < levels && l < 32; ++l) {
    if (pa[np - 1].w < 16 || pa[np - 1].h < 16) break;
    pa[np] = downsample_half(pa[np - 1]);
    pb[np] = downsample_half(pb[np - 1]);
    ++np;
  }
  const int coarsest = np - 1;
  plane u = plane_new(pa[coarsest].w, pa[coarsest].h);
  plane v = plane_new(pa[coarsest].w, pa[coarsest].h);
  for (int l = coarsest; l >= 0; --l) {
    if (l != coarsest) {
      const int w = pa[l].w, h = pa[l].h;
      const float sx = (float)w / (float)u.w;
      plane nu = resize_bilinear(u, w, h, sx);
      plane nv = resize_bilinear(v, w, h, sx);
      free(u.p);
      free(v.p);
      u = nu;
      v = nv;
    }
    refine_level(pa[l], pb[l], &u, &v, iterations, smoothness, threads);
  }
  for (int y = 0; y < ra->height; ++y)
    for (int x = 0; x < ra->width; ++x) {
      const size_t i = (size_t)y * ra->width + x;
      if (!valid_at(ra, x, y) || !valid_at(rb, x, y)) {
        uo[i] = 0.0f;
        vo[i] = 0.0f;
      } else {
        uo[i] = u.p[i];
        vo[i] = v.p[i];
      }
    }
  free(u.p);
  free(v.p);
  for (int l = 0; l < np; ++l) {
    free(pa[l].p);
    free(pb[l].p);
  }
  return SO_OK;
}

/* chamfer_distance, flow.cpp:192-223 */
static void chamfer_distance(const uint8_t* zone, int w, int h, float* d) {
  for (size_t i = 0; i < (size_t)w * h; ++i) d[i] = zone[i] ? 0.0f : SO_FAR_AWAY;
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      float best = d[(size_t)y * w + x];
      if (x > 0) best = fminf(best, d[(size_t)y * w + x - 1] + 3.0f);
      if (y > 0) {
        best = fminf(best, d[(size_t)(y - 1) * w + x] + 3.0f);
        if (x > 0) best = fminf(best, d[(size_t)(y - 1) * w + x - 1] + 4.0f);
        if (x + 1 < w) best = fminf(best, d[(size_t)(y - 1) * w + x + 1] + 4.0f);
      }
      d[(size_t)y * w + x] = best;
    }
  for (int y = h - 1; y >= 0; --y)
    for (int x = w - 1; x >= 0; --x) {
      float best = d[(size_t)y * w + x];
      if (x + 1 < w) best = fminf(best, d[(size_t)y * w + x + 1] + 3.0f);
      if (y + 1 < h) {
        best = fminf(best, d[(size_t)(y + 1) * w + x] + 3.0f);
        if (x + 1 < w) best = fminf(best, d[(size_t)(y + 1) * w + x + 1] + 4.0f);
        if (x > 0) best = fminf(best, d[(size_t)(y + 1) * w + x - 1] + 4.0f);
      }
      d[(size_t)y * w + x] = best;
    }
}

/* blend_weights, flow.cpp:227-280 */
void so_blend_weights(const so_frame* wi, const so_frame* wj, so_region bnd,
                      float* theta_i, float* theta_j) {
  const int w = wi->width, h = wi->height;
  uint8_t* ei = (uint8_t*)calloc((size_t)w * h + 1, 1);
  uint8_t* ej = (uint8_t*)calloc((size_t)w * h + 1, 1);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const int vi = valid_at(wi, x, y), vj = valid_at(wj, x, y);
      ei[(size_t)y * w + x] = vi && !vj;
      ej[(size_t)y * w + x] = vj && !vi;
    }
  float* to_j = (float*)malloc(sizeof(float) * ((size_t)w * h + 1));
  float* to_i = (float*)malloc(sizeof(float) * ((size_t)w * h + 1));
  chamfer_distance(ej, w, h, to_j);
  chamfer_distance(ei, w, h, to_i);
  const int bw = bnd.x1 - bnd.x0, bh = bnd.y1 - bnd.y0;
  for (int y = 0; y < bh; ++y)
    for (int x = 0; x < bw; ++x) {
      const float cj = to_j[(size_t)(bnd.y0 + y) * w + bnd.x0 + x];
      const float ci = to_i[(size_t)(bnd.y0 + y) * w + bnd.x0 + x];
      const float di = cj >= SO_FAR_AWAY ? SO_FAR_AWAY : fmaxf(0.0f, cj / 3.0f - 1.0f);
      const float dj = ci >= SO_FAR_AWAY ? SO_FAR_AWAY : fmaxf(0.0f, ci / 3.0f - 1.0f);
      float ti;
      if (di >= SO_FAR_AWAY && dj >= SO_FAR_AWAY)
        ti = 0.5f;
      else if (di >= SO_FAR_AWAY)
        ti = 1.0f;
      else if (dj >= SO_FAR_AWAY)
        ti = 0.0f;
      else if (di + dj <= 0.0f)
        ti = 0.5f;
      else
        ti = di / (di + dj);
      theta_i[(size_t)y * bw + x] = ti;
      if (theta_j) theta_j[(size_t)y * bw + x] = 1.0f - ti;
    }
  free(ei);
  free(ej);
  free(to_i);
  free(to_j);
}

/* flow_fuse, flow.cpp:282-322 */
int so_flow_fuse(const so_frame* ri, const so_frame* rj, const float* uij,
                 const float* vij, const float* uji, const float* vji,
                 const float* theta_i, const float* theta_j, int weighting,
                 so_frame* out) {
  const int w = ri->width, h = ri->height;
  if (rj->width != w || rj->height != h) return SO_ShapeMismatch;
  frame_alloc(out, w, h, 1, 0);
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const size_t i = (size_t)y * w + x;
      const float ti = theta_i[i];
      const float tj = theta_j[i];
      const float wi = weighting == 0 ? ti : tj;
      const float wj = weighting == 0 ? tj : ti;
      float si[3], sj[3];
      const int vi = so_sample_bilinear(ri, (double)((float)x + wi * uij[i]),
                                        (double)((float)y + wi * vij[i]), si);
      const int vj = so_sample_bilinear(rj, (double)((float)x + wj * uji[i]),
                                        (double)((float)y + wj * vji[i]), sj);
      if (!vi && !vj) continue;
      float rgb[3];
      for (int c = 0; c < 3; ++c) {
        if (vi && vj)
          rgb[c] = ti * si[c] + tj * sj[c];
        else if (vi)
          rgb[c] = si[c];
        else
          rgb[c] = sj[c];
      }
      uint8_t* p = out->data + i * 3;
      p[0] = so_quantize_channel(rgb[0]);
      p[1] = so_quantize_channel(rgb[1]);
      p[2] = so_quantize_channel(rgb[2]);
      out->mask[i] = 1;
    }
  return SO_OK;
}

/* compose_panorama, flow.cpp:324-357 */
int so_compose_panorama(const so_frame* wi, const so_frame* wj,
                        const so_frame* fused, so_region ov, so_frame* out) {
  if (wi->width != wj->width || wi->height != wj->height) return SO_ShapeMismatch;
  frame_alloc(out, wi->width, wi->height, 1, 0);
  for (int y = 0; y < out->height; ++y)
    for (int x = 0; x < out->width; ++x) {
      const int vi = valid_at(wi, x, y), vj = valid_at(wj, x, y);
      const uint8_t* src = NULL;
      if (vi && vj) {
        const int dx = x - ov.x0, dy = y - ov.y0;
        if (valid_at(fused, dx, dy))
          src = px(fused, dx, dy);
        else
          src = px(wi, x, y);
      } else if (vi) {
        src = px(wi, x, y);
      } else if (vj) {
        src = px(wj, x, y);
      }
      if (!src) continue;
      uint8_t* d = out->data + ((size_t)y * out->width + x) * 3;
      d[0] = src[0];
      d[1] = src[1];
      d[2] = src[2];
      out->mask[(size_t)y * out->width + x] = 1;
    }
  return SO_OK;
}

/* ------------------------------------------------------------------------ */
/* Pipeline: pipeline.hpp:47-63, pipeline.cpp:209-360                         */
/* ------------------------------------------------------------------------ */

typedef struct {
  int view, partner;
  so_region bounds;
  float* theta_i;
  float* theta_j;
  so_window window;
} so_pair;

struct so_state {
  so_config cfg;
  int canvas_w, canvas_h;
  double offx, offy;
  double* lsin;  /* cylindrical lift tables (NULL: planar) */
  double* lcos;
  double* lh;
  double maps[SO_MAX_VIEWS][9];
  double inv[SO_MAX_VIEWS][9];
  so_region view_bbox[SO_MAX_VIEWS];
  int n_pairs;
  so_pair pairs[SO_MAX_VIEWS];
  int hist_n;
  int hist_m1[3][3], hist_m2[3][3];
  long frame_counter;
  /* debug intermediates of the last frame */
  so_frame dbg_warped[SO_MAX_VIEWS];
  float* dbg_flow[SO_MAX_VIEWS][2][2];
  int refine_warning[SO_MAX_VIEWS];
};

static int effective_topology(const so_config* c) {
  if (c->topology == 1 || c->topology == 2) return c->topology;
  return c->n_views <= 3 ? 1 : 2;
}

/* Pair construction.  Star (pipeline.cpp:233-239): every non-reference view
 * in ascending order, partner = reference.  Chain (N-view extension):
 * partner = neighbour toward the reference, pairs ordered by distance from
 * the reference then by index, so a partner is always corrected first. */
static void build_pairs(so_state* s) {
  const so_config* c = &s->cfg;
  const int topo = (c->topology == 3 || (c->topology == 0 && c->projection == 1))
                       ? 3 : effective_topology(c);
  s->n_pairs = 0;
  if (topo == 3) {
    /* ring chain: k = (v - ref) mod N, distance min(k, N - k), partner one
     * step toward the reference (the k = N/2 view pairs with k - 1) */
    const int n = c->n_views;
    for (int d = 1; d <= n / 2; ++d)
      for (int v = 0; v < n; ++v) {
        const int k = ((v - c->reference) % n + n) % n;
        if ((k < n - k ? k : n - k) != d) continue;
        s->pairs[s->n_pairs].view = v;
        s->pairs[s->n_pairs].partner = (k <= n / 2) ? (v - 1 + n) % n : (v + 1) % n;
        s->n_pairs++;
      }
    return;
  }
  if (topo == 1) {
    for (int v = 0; v < c->n_views; ++v) {
      if (v == c->reference) continue;
      s->pairs[s->n_pairs].view = v;
      s->pairs[s->n_pairs].partner = c->reference;
      s->n_pairs++;
    }
    return;
  }
  for (int d = 1; d < c->n_views; ++d)
    for (int v = 0; v < c->n_views; ++v) {
      if (abs(v - c->reference) != d) continue;
      s->pairs[s->n_pairs].view = v;
      s->pairs[s->n_pairs].partner = v < c->reference ? v + 1 : v - 1;
      s->n_pairs++;
    }
}

/* initialize, pipeline.cpp:209-257, with refinement disabled (the
 * per-frame path's configs use fixed/coarse homographies).  Masks depend
 * only on geometry for unmasked inputs, so a zero frame is warped. */
/* rebuild_pair_geometry (pipeline.cpp:181-205): warp masks (geometry only:
 * the warped pixel values are not needed), view footprints, overlap bounds
 * and blend weights of every pair. */
/* With first frames that carry masks (frame.hpp:44-47), the pair bounds and
 * blend weights come from the warps of those frames, as the reference's
 * rebuild_pair_geometry warps first_frames; the view footprints stay the
 * geometry-only ones (a superset of any frame's warp). */
static int rebuild_pair_geometry_frames(so_state* s, const so_frame* first) {
  const so_config* cfg = &s->cfg;
  so_frame warped[SO_MAX_VIEWS];
  for (int v = 0; v < cfg->n_views; ++v) {
    so_frame zero;
    frame_alloc(&zero, cfg->width[v], cfg->height[v], 0, 0);
    int e = so_warp_frame_lift(&zero, s->inv[v], s->canvas_w, s->canvas_h, s->offx,
                               s->offy, s->lsin, s->lcos, s->lh, cfg->threads, &warped[v]);
    so_free_frame(&zero);
    if (e == SO_OK) mask_bbox(&warped[v], &s->view_bbox[v]);
    if (e == SO_OK && first && first[v].mask) {
      so_free_frame(&warped[v]);
      e = so_warp_frame_lift(&first[v], s->inv[v], s->canvas_w, s->canvas_h, s->offx,
                             s->offy, s->lsin, s->lcos, s->lh, cfg->threads, &warped[v]);
    }
    if (e != SO_OK) {
      for (int u = 0; u < v; ++u) so_free_frame(&warped[u]);
      return e;
    }
  }
  for (int k = 0; k < s->n_pairs; ++k) {
    so_pair* p = &s->pairs[k];
    int e = overlap_bounds(&warped[p->view], &warped[p->partner], &p->bounds);
    if (e != SO_OK) {
      for (int u = 0; u < cfg->n_views; ++u) so_free_frame(&warped[u]);
      for (int q = 0; q < k; ++q) {
        free(s->pairs[q].theta_i);
        free(s->pairs[q].theta_j);
        s->pairs[q].theta_i = s->pairs[q].theta_j = NULL;
      }
      return (e == SO_NoOverlap) ? SO_ConfigurationError : e;
    }
    const size_t n = (size_t)(p->bounds.x1 - p->bounds.x0) *
                     (p->bounds.y1 - p->bounds.y0);
    p->theta_i = (float*)malloc(sizeof(float) * n);
    p->theta_j = (float*)malloc(sizeof(float) * n);
    so_blend_weights(&warped[p->view], &warped[p->partner], p->bounds,
                     p->theta_i, p->theta_j);
  }
  for (int v = 0; v < cfg->n_views; ++v) so_free_frame(&warped[v]);
  return SO_OK;
}

static int rebuild_pair_geometry(so_state* s) { return rebuild_pair_geometry_frames(s, NULL); }

static int any_mask(const so_frame* first, int n) {
  if (!first) return 0;
  for (int v = 0; v < n; ++v)
    if (first[v].mask) return 1;
  return 0;
}

so_state* so_initialize(const so_config* cfg, int* err) {
  *err = SO_OK;
  if (cfg->n_views < 2 || cfg->n_views > SO_MAX_VIEWS || cfg->reference < 0 ||
      cfg->reference >= cfg->n_views) {
    *err = SO_ConfigurationError;
    return NULL;
  }
  so_state* s = (so_state*)calloc(1, sizeof(so_state));
  s->cfg = *cfg;
  int wc = cfg->window_capacity;
  if (wc < 1) wc = 1;
  if (wc > 3) wc = 3;
  if (cfg->projection == 1) {
    /* cylindrical 360-degree canvas (extension): A_v = K_v R_v R_ref^T */
    const double f = cfg->cyl_focal > 0.0 ? cfg->cyl_focal : cfg->cams[cfg->reference].fx;
    s->cfg.cyl_focal = f;
    double rref[9], rrefT[9];
    memcpy(rref, cfg->cams[cfg->reference].rotation, sizeof(rref));
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) rrefT[i * 3 + j] = rref[j * 3 + i];
    double hmin = DBL_MAX, hmax = -DBL_MAX;
    for (int v = 0; v < cfg->n_views; ++v) {
      const so_camera* c = &cfg->cams[v];
      const double k[9] = {c->fx, 0, c->cx, 0, c->fy, c->cy, 0, 0, 1};
      double kr[9], rT[9], m[9];
      mul3(k, c->rotation, kr);
      mul3(kr, rrefT, s->inv[v]);
      for (int i = 0; i < 9; ++i) s->maps[v][i] = s->inv[v][i];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) rT[i * 3 + j] = c->rotation[j * 3 + i];
      mul3(rref, rT, m); /* camera v -> reference frame */
      const int W = cfg->width[v], H = cfg->height[v];
      for (int e2 = 0; e2 < 2; ++e2) {
        const int count = e2 == 0 ? W : H;
        for (int i = 0; i < count; ++i)
          for (int side = 0; side < 2; ++side) {
            const double px = e2 == 0 ? (double)i : (side ? W - 1.0 : 0.0);
            const double py = e2 == 0 ? (side ? H - 1.0 : 0.0) : (double)i;
            const double cx = (px - c->cx) / c->fx, cy = (py - c->cy) / c->fy;
            const double rx = (m[0] * cx + m[1] * cy) + m[2];
            const double ry = (m[3] * cx + m[4] * cy) + m[5];
            const double rz = (m[6] * cx + m[7] * cy) + m[8];
            const double hh = ry / sqrt(rx * rx + rz * rz);
            hmin = fmin(hmin, hh);
            hmax = fmax(hmax, hh);
          }
      }
    }
    s->canvas_w = (int)ceil(2.0 * M_PI * f);
    s->offx = -floor(s->canvas_w / 2.0);
    s->offy = floor(hmin * f);
    s->canvas_h = (int)(ceil(hmax * f) - s->offy) + 1;
    s->lsin = (double*)malloc(sizeof(double) * s->canvas_w);
    s->lcos = (double*)malloc(sizeof(double) * s->canvas_w);
    s->lh = (double*)malloc(sizeof(double) * s->canvas_h);
    for (int x = 0; x < s->canvas_w; ++x) {
      const double t = (x + s->offx) / f;
      s->lsin[x] = sin(t);
      s->lcos[x] = cos(t);
    }
    for (int y = 0; y < s->canvas_h; ++y) s->lh[y] = (y + s->offy) / f;
  } else {
  double cam[SO_MAX_VIEWS][9];
  for (int v = 0; v < cfg->n_views; ++v) {
    int e = planar_homography(&cfg->cams[v], cam[v]);
    if (e != SO_OK) {
      *err = e;
      free(s);
      return NULL;
    }
  }
  double min_x = DBL_MAX, min_y = DBL_MAX, max_x = -DBL_MAX, max_y = -DBL_MAX;
  for (int v = 0; v < cfg->n_views; ++v) {
    int e = pairwise_homography(cam[cfg->reference], cam[v], s->maps[v]);
    if (e != SO_OK) {
      *err = e;
      free(s);
      return NULL;
    }
    so_inverse3(s->maps[v], s->inv[v]);
    /* compute_canvas, geometry.cpp:147-171 */
    const double w = cfg->width[v] - 1.0, h = cfg->height[v] - 1.0;
    const double cx[4] = {0.0, w, 0.0, w}, cy[4] = {0.0, 0.0, h, h};
    for (int k = 0; k < 4; ++k) {
      double X, Y;
      homography_apply(s->maps[v], cx[k], cy[k], &X, &Y);
      min_x = fmin(min_x, X);
      min_y = fmin(min_y, Y);
      max_x = fmax(max_x, X);
      max_y = fmax(max_y, Y);
    }
  }
  s->offx = floor(min_x);
  s->offy = floor(min_y);
  s->canvas_w = (int)(ceil(max_x) - s->offx) + 1;
  s->canvas_h = (int)(ceil(max_y) - s->offy) + 1;
  }

  build_pairs(s);
  for (int k = 0; k < s->n_pairs; ++k) {
    s->pairs[k].window.capacity = wc;
    s->pairs[k].window.size = 0;
  }
  int e = rebuild_pair_geometry(s);
  if (e != SO_OK) {
    *err = e;
    free(s->lsin);
    free(s->lcos);
    free(s->lh);
    free(s);
    return NULL;
  }
  return s;
}

/* Homography::apply with hnormalized (geometry.cpp:33-36) */
static void h_apply(const double* h, double x, double y, double* ox, double* oy) {
  const double q0 = (h[0] * x + h[1] * y) + h[2];
  const double q1 = (h[3] * x + h[4] * y) + h[5];
  const double q2 = (h[6] * x + h[7] * y) + h[8];
  *ox = q0 / q2;
  *oy = q1 / q2;
}

/* broaden (geometry.cpp:119-133) */
static so_region broaden(so_region r, double margin, so_region b) {
  const int mx = (int)lround(margin * (r.x1 - r.x0));
  const int my = (int)lround(margin * (r.y1 - r.y0));
  so_region o;
  o.x0 = r.x0 - mx > b.x0 ? r.x0 - mx : b.x0;
  o.y0 = r.y0 - my > b.y0 ? r.y0 - my : b.y0;
  o.x1 = r.x1 + mx < b.x1 ? r.x1 + mx : b.x1;
  o.y1 = r.y1 + my < b.y1 ? r.y1 + my : b.y1;
  return o;
}

/* refine_pair (pipeline.cpp:114-179) against the pair's partner (the
 * reference for the star topology): detect / describe / match on the
 * broadened overlap of the warped first frames, matches back-projected to
 * the view's source plane, RANSAC scale + translation, translation carried
 * to the plane with the local Jacobian, map := T * H * S. */
static int refine_pair(so_state* s, const so_frame* warped, int k) {
  const so_config* cfg = &s->cfg;
  so_pair* p = &s->pairs[k];
  s->refine_warning[k] = 1;
  const so_region canvas_r = {0, 0, s->canvas_w, s->canvas_h};
  const so_region search = broaden(p->bounds, cfg->refine_margin, canvas_r);
  so_keypoint *kv = NULL, *kr = NULL;
  int nv = 0, nr = 0;
  if (so_detect(&warped[p->view], search, cfg->detect_threshold, &kv, &nv) != SO_OK ||
      so_detect(&warped[p->partner], search, cfg->detect_threshold, &kr, &nr) != SO_OK ||
      nv == 0 || nr == 0) {
    free(kv);
    free(kr);
    return SO_OK;
  }
  float* dv = (float*)malloc(sizeof(float) * 64 * nv);
  float* dr = (float*)malloc(sizeof(float) * 64 * nr);
  so_describe(&warped[p->view], kv, nv, dv);
  so_describe(&warped[p->partner], kr, nr, dr);
  so_match_pair* m = (so_match_pair*)malloc(sizeof(so_match_pair) * (nv > 0 ? nv : 1));
  const int nm = so_match(dv, nv, dr, nr, kv, kr, cfg->match_ratio, m);
  const double* map = s->maps[p->view];
  double inv_raw[9], inv[9];
  so_inverse3(map, inv_raw);
  homography_from_matrix(inv_raw, inv); /* Homography::inverse, geometry.cpp:29-31 */
  for (int i = 0; i < nm; ++i) {
    double qx, qy, px, py;
    h_apply(inv, m[i].ax + s->offx, m[i].ay + s->offy, &qx, &qy);
    h_apply(inv, m[i].bx + s->offx, m[i].by + s->offy, &px, &py);
    m[i].ax = qx;
    m[i].ay = qy;
    m[i].bx = px;
    m[i].by = py;
  }
  so_similarity fit;
  const int e = so_ransac(m, nm, cfg->ransac_iters, cfg->inlier_px, 0.5, 2.0,
                          cfg->seed + (unsigned long long)p->view, &fit);
  free(kv);
  free(kr);
  free(dv);
  free(dr);
  free(m);
  if (e != SO_OK) return SO_OK; /* NoConsensus / InsufficientMatches: keep the map */
  /* centre of the overlap and local_jacobian (pipeline.cpp:98-112) */
  const double cx = s->offx + p->bounds.x0 + (p->bounds.x1 - p->bounds.x0) / 2.0;
  const double cy = s->offy + p->bounds.y0 + (p->bounds.y1 - p->bounds.y0) / 2.0;
  double ax, ay;
  h_apply(inv, cx, cy, &ax, &ay);
  const double eps = 1e-4;
  double xp0, yp0, xm0, ym0, xp1, yp1, xm1, ym1;
  h_apply(map, ax + eps, ay, &xp0, &yp0);
  h_apply(map, ax - eps, ay, &xm0, &ym0);
  h_apply(map, ax, ay + eps, &xp1, &yp1);
  h_apply(map, ax, ay - eps, &xm1, &ym1);
  const double j00 = (xp0 - xm0) / (2 * eps), j10 = (yp0 - ym0) / (2 * eps);
  const double j01 = (xp1 - xm1) / (2 * eps), j11 = (yp1 - ym1) / (2 * eps);
  const double tx = j00 * fit.t_x + j01 * fit.t_y;
  const double ty = j10 * fit.t_x + j11 * fit.t_y;
  /* refine_homography (geometry.cpp:135-145): T(tx, ty) * H * S(sx, sy) */
  const double t[9] = {1, 0, tx, 0, 1, ty, 0, 0, 1};
  const double sc[9] = {fit.s_x, 0, 0, 0, fit.s_y, 0, 0, 0, 1};
  double th[9], ths[9];
  mul3(t, map, th);
  mul3(th, sc, ths);
  double refined[9];
  const int fe = homography_from_matrix(ths, refined);
  if (fe != SO_OK) return fe; /* SingularHomography propagates (pipeline.cpp:171-177) */
  memcpy(s->maps[p->view], refined, sizeof(refined));
  so_inverse3(s->maps[p->view], s->inv[p->view]); /* pipeline.cpp:40 */
  s->refine_warning[k] = 0;
  return SO_OK;
}

static void free_pair_weights(so_state* s) {
  for (int k = 0; k < s->n_pairs; ++k) {
    free(s->pairs[k].theta_i);
    free(s->pairs[k].theta_j);
    s->pairs[k].theta_i = s->pairs[k].theta_j = NULL;
  }
}

so_state* so_initialize_frames(const so_config* cfg, const so_frame* first, int* err) {
  so_state* s = so_initialize(cfg, err);
  if (!s || !first) return s;
  if (any_mask(first, cfg->n_views)) {
    /* masked first frames: the pair geometry of their warps (pipeline.cpp:246) */
    free_pair_weights(s);
    const int e = rebuild_pair_geometry_frames(s, first);
    if (e != SO_OK) {
      so_destroy(s);
      *err = e;
      return NULL;
    }
  }
  if (!cfg->refine_enabled) return s;
  if (cfg->projection == 1) return s; /* refinement serves the planar canvas */
  so_frame warped[SO_MAX_VIEWS];
  for (int v = 0; v < cfg->n_views; ++v) {
    const int e = so_warp_frame(&first[v], s->inv[v], s->canvas_w, s->canvas_h, s->offx, s->offy,
                                cfg->threads, &warped[v]);
    if (e != SO_OK) {
      for (int u = 0; u < v; ++u) so_free_frame(&warped[u]);
      so_destroy(s);
      *err = e;
      return NULL;
    }
  }
  int re = SO_OK;
  for (int k = 0; k < s->n_pairs && re == SO_OK; ++k) re = refine_pair(s, warped, k);
  for (int v = 0; v < cfg->n_views; ++v) so_free_frame(&warped[v]);
  if (re != SO_OK) {
    so_destroy(s);
    *err = re;
    return NULL;
  }
  /* refinement moved the maps: bounds and weights shift (pipeline.cpp:254) */
  free_pair_weights(s);
  const int e = rebuild_pair_geometry_frames(s, first);
  if (e != SO_OK) {
    so_destroy(s);
    *err = e;
    return NULL;
  }
  return s;
}

int so_state_refine_warning(const so_state* s, int k) { return s->refine_warning[k]; }

void so_destroy(so_state* s) {
  if (!s) return;
  for (int k = 0; k < s->n_pairs; ++k) {
    free(s->pairs[k].theta_i);
    free(s->pairs[k].theta_j);
    window_free(&s->pairs[k].window);
    for (int d = 0; d < 2; ++d)
      for (int c = 0; c < 2; ++c) free(s->dbg_flow[k][d][c]);
  }
  for (int v = 0; v < SO_MAX_VIEWS; ++v) so_free_frame(&s->dbg_warped[v]);
  free(s->lsin);
  free(s->lcos);
  free(s->lh);
  free(s);
}

/* process_frame, pipeline.cpp:259-360 */
int so_process_frame(so_state* s, const so_frame* frames, so_frame* pano_out,
                     so_report* rep) {
  const so_config* cfg = &s->cfg;
  const int nv = cfg->n_views;
  const int nt = cfg->threads > 0 ? cfg->threads : 1;
  memset(rep, 0, sizeof(*rep));
  rep->frame_index = s->frame_counter;
  rep->n_pairs = s->n_pairs;
  for (int v = 0; v < nv; ++v)
    if (frames[v].width != cfg->width[v] || frames[v].height != cfg->height[v])
      return SO_InputMismatch;

  /* Geometric warping (pipeline.cpp:270-277) */
  double t0 = now_seconds();
  so_frame warped[SO_MAX_VIEWS];
  for (int v = 0; v < nv; ++v) {
    int e = so_warp_frame_lift(&frames[v], s->inv[v], s->canvas_w, s->canvas_h,
                               s->offx, s->offy, s->lsin, s->lcos, s->lh, nt, &warped[v]);
    if (e != SO_OK) {
      for (int u = 0; u <= v; ++u) so_free_frame(&warped[u]);
      return e;
    }
    if (cfg->keep_debug) {
      so_free_frame(&s->dbg_warped[v]);
      frame_copy(&s->dbg_warped[v], &warped[v]);
    }
  }
  rep->stage_seconds[0] = now_seconds() - t0;

  /* Color correction (pipeline.cpp:279-300) */
  t0 = now_seconds();
  for (int k = 0; k < s->n_pairs; ++k) {
    so_pair* p = &s->pairs[k];
    double m[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    int rank_def = 0;
    int e = transfer_step(&warped[p->view], &warped[p->partner], p->bounds,
                          &p->window, m, &rank_def);
    int degraded = rank_def;
    if (e != SO_OK) {
      for (int i = 0; i < 9; ++i) m[i] = (i % 4 == 0) ? 1.0 : 0.0;
      degraded = 1;
    }
    so_apply_color_matrix_rows(&warped[p->view], m, nt);
    memcpy(rep->m[k], m, sizeof(m));
    rep->rank_deficient[k] = degraded;
  }
  rep->stage_seconds[1] = now_seconds() - t0;

  /* Local warping (pipeline.cpp:302-322) */
  t0 = now_seconds();
  so_frame crop_v[SO_MAX_VIEWS], crop_r[SO_MAX_VIEWS];
  float* fl[SO_MAX_VIEWS][4];
  for (int k = 0; k < s->n_pairs; ++k) {
    so_pair* p = &s->pairs[k];
    crop_frame(&warped[p->view], p->bounds, &crop_v[k]);
    crop_frame(&warped[p->partner], p->bounds, &crop_r[k]);
    const size_t n = (size_t)crop_v[k].width * crop_v[k].height;
    for (int j = 0; j < 4; ++j) fl[k][j] = (float*)calloc(n + 1, sizeof(float));
    int e = so_dense_flow(&crop_v[k], &crop_r[k], cfg->flow_levels,
                          cfg->flow_iterations, cfg->smoothness, nt, fl[k][0],
                          fl[k][1]);
    if (e == SO_OK)
      e = so_dense_flow(&crop_r[k], &crop_v[k], cfg->flow_levels,
                        cfg->flow_iterations, cfg->smoothness, nt, fl[k][2],
                        fl[k][3]);
    if (e != SO_OK)
      for (int j = 0; j < 4; ++j) memset(fl[k][j], 0, n * sizeof(float));
    if (cfg->keep_debug) {
      for (int d = 0; d < 2; ++d)
        for (int c = 0; c < 2; ++c) {
          free(s->dbg_flow[k][d][c]);
          s->dbg_flow[k][d][c] = (float*)malloc(n * sizeof(float) + 4);
          memcpy(s->dbg_flow[k][d][c], fl[k][d * 2 + c], n * sizeof(float));
        }
    }
  }
  rep->stage_seconds[2] = now_seconds() - t0;

  /* Image blending (pipeline.cpp:324-334) */
  t0 = now_seconds();
  so_frame pano;
  frame_copy(&pano, &warped[cfg->reference]);
  for (int k = 0; k < s->n_pairs; ++k) {
    so_pair* p = &s->pairs[k];
    so_frame fused, next;
    so_flow_fuse(&crop_v[k], &crop_r[k], fl[k][0], fl[k][1], fl[k][2],
                 fl[k][3], p->theta_i, p->theta_j, cfg->fuse_weighting, &fused);
    so_compose_panorama(&pano, &warped[p->view], &fused, p->bounds, &next);
    so_free_frame(&pano);
    so_free_frame(&fused);
    pano = next;
  }
  rep->stage_seconds[3] = now_seconds() - t0;

  /* Global balancing (pipeline.cpp:336-355) */
  t0 = now_seconds();
  so_hist hist;
  const so_region full = {0, 0, pano.width, pano.height};
  if (so_compute_histogram(&pano, full, &hist) == SO_OK) {
    int m1[3], m2[3];
    if (so_find_thresholds(&hist, cfg->lambda, m1, m2) == SO_OK) {
      if (s->hist_n == 3) {
        memmove(s->hist_m1[0], s->hist_m1[1], sizeof(int) * 6);
        memmove(s->hist_m2[0], s->hist_m2[1], sizeof(int) * 6);
        s->hist_n = 2;
      }
      memcpy(s->hist_m1[s->hist_n], m1, sizeof(m1));
      memcpy(s->hist_m2[s->hist_n], m2, sizeof(m2));
      s->hist_n++;
      int sm1[3], sm2[3];
      so_smooth_thresholds(s->hist_n, (const int(*)[3])s->hist_m1,
                           (const int(*)[3])s->hist_m2, sm1, sm2);
      uint8_t lut[3][256];
      if (so_build_curve(sm1, sm2, cfg->gamma_dark, cfg->gamma_bright,
                         cfg->target_black, cfg->target_white, lut) == SO_OK) {
        /* apply_tone_rows, pipeline.cpp:84-96 */
#pragma omp parallel for schedule(static) num_threads(nt)
        for (int y = 0; y < pano.height; ++y)
          for (int x = 0; x < pano.width; ++x) {
            if (!valid_at(&pano, x, y)) continue;
            uint8_t* q = pano.data + ((size_t)y * pano.width + x) * 3;
            q[0] = lut[0][q[0]];
            q[1] = lut[1][q[1]];
            q[2] = lut[2][q[2]];
          }
        memcpy(rep->threshold_m1, sm1, sizeof(sm1));
        memcpy(rep->threshold_m2, sm2, sizeof(sm2));
        rep->balanced = 1;
      }
    }
  }
  rep->stage_seconds[1] += now_seconds() - t0;

  ++s->frame_counter;
  for (int k = 0; k < s->n_pairs; ++k) {
    so_free_frame(&crop_v[k]);
    so_free_frame(&crop_r[k]);
    for (int j = 0; j < 4; ++j) free(fl[k][j]);
  }
  for (int v = 0; v < nv; ++v) so_free_frame(&warped[v]);
  *pano_out = pano;
  return SO_OK;
}

/* ---- inspection ---- */
void so_state_canvas(const so_state* s, int* w, int* h, double* offx,
                     double* offy) {
  *w = s->canvas_w;
  *h = s->canvas_h;
  *offx = s->offx;
  *offy = s->offy;
}

void so_state_map(const so_state* s, int view, double h[9], double inv[9]) {
  memcpy(h, s->maps[view], sizeof(double) * 9);
  memcpy(inv, s->inv[view], sizeof(double) * 9);
}

int so_state_n_pairs(const so_state* s) { return s->n_pairs; }

void so_state_pair(const so_state* s, int k, int* view, int* partner,
                   so_region* bounds) {
  *view = s->pairs[k].view;
  *partner = s->pairs[k].partner;
  *bounds = s->pairs[k].bounds;
}

void so_state_pair_weights(const so_state* s, int k, float* theta_i) {
  const so_region b = s->pairs[k].bounds;
  memcpy(theta_i, s->pairs[k].theta_i,
         sizeof(float) * (size_t)(b.x1 - b.x0) * (b.y1 - b.y0));
}

void so_state_view_bbox(const so_state* s, int view, so_region* bbox) {
  *bbox = s->view_bbox[view];
}

int so_state_last_flow(const so_state* s, int k, int dir, float* u, float* v) {
  if (!s->dbg_flow[k][dir][0]) return SO_MissingState;
  const so_region b = s->pairs[k].bounds;
  const size_t n = (size_t)(b.x1 - b.x0) * (b.y1 - b.y0);
  memcpy(u, s->dbg_flow[k][dir][0], n * sizeof(float));
  memcpy(v, s->dbg_flow[k][dir][1], n * sizeof(float));
  return SO_OK;
}

int so_state_last_warped(const so_state* s, int view, uint8_t* rgb,
                         uint8_t* mask) {
  const so_frame* f = &s->dbg_warped[view];
  if (!f->data) return SO_MissingState;
  memcpy(rgb, f->data, (size_t)f->width * f->height * 3);
  memcpy(mask, f->mask, (size_t)f->width * f->height);
  return SO_OK;
}

/* ======================================================================
 * Quality metrics (metrics.cpp:9-155)
 * ====================================================================== */

static int so_valid(const so_frame* f, int x, int y) {
  return f->mask == NULL || f->mask[(size_t)y * f->width + x] != 0;
}

/* psnr, metrics.cpp:9-31 */
int so_psnr(const so_frame* a, const so_frame* b, double* out) {
  if (a->width != b->width || a->height != b->height) return SO_ShapeMismatch;
  long long n = 0;
  double sse = 0.0;
  for (int y = 0; y < a->height; ++y)
    for (int x = 0; x < a->width; ++x) {
      if (!so_valid(a, x, y) || !so_valid(b, x, y)) continue;
      const uint8_t* pa = a->data + ((size_t)y * a->width + x) * 3;
      const uint8_t* pb = b->data + ((size_t)y * b->width + x) * 3;
      for (int c = 0; c < 3; ++c) {
        const double d = (double)pa[c] - pb[c];
        sse += d * d;
      }
      ++n;
    }
  if (n == 0) return SO_EmptyRegion;
  const double mse = sse / (3.0 * (double)n);
  *out = mse == 0.0 ? INFINITY : 10.0 * log10(255.0 * 255.0 / mse);
  return SO_OK;
}

#define SO_SSIM_WIN 11

/* gaussian_kernel, metrics.cpp:40-49 */
static void so_gauss_kernel(double k[SO_SSIM_WIN]) {
  double sum = 0.0;
  for (int i = 0; i < SO_SSIM_WIN; ++i) {
    const double d = i - (SO_SSIM_WIN - 1) / 2.0;
    k[i] = exp(-d * d / (2.0 * 1.5 * 1.5));
    sum += k[i];
  }
  for (int i = 0; i < SO_SSIM_WIN; ++i) k[i] /= sum;
}

/* gauss_filter, metrics.cpp:56-79: horizontal then vertical, interior only */
static void so_gauss_filter(const double* src, int w, int h, double* out) {
  double k[SO_SSIM_WIN];
  so_gauss_kernel(k);
  const int r = SO_SSIM_WIN / 2;
  double* tmp = (double*)calloc((size_t)w * h, sizeof(double));
  for (int y = 0; y < h; ++y)
    for (int x = r; x < w - r; ++x) {
      double acc = 0.0;
      for (int i = 0; i < SO_SSIM_WIN; ++i) acc += k[i] * src[(size_t)y * w + x - r + i];
      tmp[(size_t)y * w + x] = acc;
    }
  memset(out, 0, sizeof(double) * (size_t)w * h);
  for (int y = r; y < h - r; ++y)
    for (int x = 0; x < w; ++x) {
      double acc = 0.0;
      for (int i = 0; i < SO_SSIM_WIN; ++i) acc += k[i] * tmp[(size_t)(y - r + i) * w + x];
      out[(size_t)y * w + x] = acc;
    }
  free(tmp);
}

/* ssim, metrics.cpp:83-155 */
int so_ssim(const so_frame* a, const so_frame* b, double* out) {
  if (a->width != b->width || a->height != b->height) return SO_ShapeMismatch;
  if (a->width < SO_SSIM_WIN || a->height < SO_SSIM_WIN) return SO_TooSmall;
  const int w = a->width, h = a->height;
  const size_t n = (size_t)w * h;
  double* la = (double*)malloc(sizeof(double) * n);
  double* lb = (double*)malloc(sizeof(double) * n);
  double* sq = (double*)malloc(sizeof(double) * n);
  double* mu_a = (double*)malloc(sizeof(double) * n);
  double* mu_b = (double*)malloc(sizeof(double) * n);
  double* aa = (double*)malloc(sizeof(double) * n);
  double* bb = (double*)malloc(sizeof(double) * n);
  double* ab = (double*)malloc(sizeof(double) * n);
  uint8_t* joint = (uint8_t*)malloc(n);
  uint32_t* integ = (uint32_t*)calloc((size_t)(w + 1) * (h + 1), sizeof(uint32_t));
  for (int y = 0; y < h; ++y)
    for (int x = 0; x < w; ++x) {
      const size_t i = (size_t)y * w + x;
      const int valid = so_valid(a, x, y) && so_valid(b, x, y);
      joint[i] = (uint8_t)valid;
      const uint8_t* pa = a->data + i * 3;
      const uint8_t* pb = b->data + i * 3;
      la[i] = valid ? 0.299 * pa[0] + 0.587 * pa[1] + 0.114 * pa[2] : 0.0;
      lb[i] = valid ? 0.299 * pb[0] + 0.587 * pb[1] + 0.114 * pb[2] : 0.0;
    }
  for (int y = 0; y < h; ++y) {
    uint32_t row = 0;
    for (int x = 0; x < w; ++x) {
      row += joint[(size_t)y * w + x];
      integ[(size_t)(y + 1) * (w + 1) + x + 1] = integ[(size_t)y * (w + 1) + x + 1] + row;
    }
  }
  so_gauss_filter(la, w, h, mu_a);
  so_gauss_filter(lb, w, h, mu_b);
  for (size_t i = 0; i < n; ++i) sq[i] = la[i] * la[i];
  so_gauss_filter(sq, w, h, aa);
  for (size_t i = 0; i < n; ++i) sq[i] = lb[i] * lb[i];
  so_gauss_filter(sq, w, h, bb);
  for (size_t i = 0; i < n; ++i) sq[i] = la[i] * lb[i];
  so_gauss_filter(sq, w, h, ab);
  const double c1 = (0.01 * 255.0) * (0.01 * 255.0);
  const double c2 = (0.03 * 255.0) * (0.03 * 255.0);
  const int r = SO_SSIM_WIN / 2;
  double sum = 0.0;
  long long count = 0;
  for (int y = r; y < h - r; ++y)
    for (int x = r; x < w - r; ++x) {
      const int x0 = x - r, y0 = y - r, x1 = x + r + 1, y1 = y + r + 1;
      const uint32_t cnt = integ[(size_t)y1 * (w + 1) + x1] - integ[(size_t)y0 * (w + 1) + x1] -
                           integ[(size_t)y1 * (w + 1) + x0] + integ[(size_t)y0 * (w + 1) + x0];
      if (cnt != (uint32_t)(SO_SSIM_WIN * SO_SSIM_WIN)) continue;
      const size_t i = (size_t)y * w + x;
      const double ma = mu_a[i], mb = mu_b[i];
      const double va = aa[i] - ma * ma;
      const double vb = bb[i] - mb * mb;
      const double cov = ab[i] - ma * mb;
      const double num = (2.0 * ma * mb + c1) * (2.0 * cov + c2);
      const double den = (ma * ma + mb * mb + c1) * (va + vb + c2);
      sum += num / den;
      ++count;
    }
  free(la); free(lb); free(sq); free(mu_a); free(mu_b); free(aa); free(bb); free(ab);
  free(joint); free(integ);
  if (count == 0) return SO_EmptyRegion;
  *out = sum / (double)count;
  return SO_OK;
}
