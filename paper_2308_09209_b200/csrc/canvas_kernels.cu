// canvas_kernels.cu -- geometric warping (overlap crops), the canvas pass
// (warp + colour matrix + flow fusion + composition + histogram + global
// balance LUT) and the tone/output pass.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "device_math.cuh"
#include "kernels.cuh"

namespace stitch_b200_dev {

// ---------------------------------------------------------------------------
// RGB8 -> RGBA8 expansion of the camera frames (one 32-bit load per
// bilinear neighbour downstream).  4 pixels per thread: three aligned 32-bit
// loads, one 16-byte store.  grid: (x blocks, views)
// ---------------------------------------------------------------------------
// alpha: the frame's mask byte normalised to 0/1 (Frame::mask, frame.hpp:44-47),
// 1 for an unmasked frame; only the masked samplers read it.
__device__ __forceinline__ void expand_span(const std::uint8_t* __restrict__ src,
                                            const std::uint8_t* __restrict__ mask,
                                            uchar4* __restrict__ dst, long long n) {
  const long long n4 = n / 4;
  const unsigned int* s4 = reinterpret_cast<const unsigned int*>(src);
  const unsigned int* m4 = reinterpret_cast<const unsigned int*>(mask);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const unsigned int w0 = __ldg(s4 + 3 * i), w1 = __ldg(s4 + 3 * i + 1),
                       w2 = __ldg(s4 + 3 * i + 2);
    unsigned int a0 = 1u, a1 = 1u, a2 = 1u, a3 = 1u;
    if (mask) {
      const unsigned int m = __ldg(m4 + i);
      a0 = (m & 0xffu) != 0u;
      a1 = (m & 0xff00u) != 0u;
      a2 = (m & 0xff0000u) != 0u;
      a3 = (m & 0xff000000u) != 0u;
    }
    uint4 o;
    o.x = (w0 & 0x00ffffffu) | (a0 << 24);
    o.y = (w0 >> 24) | ((w1 & 0x0000ffffu) << 8) | (a1 << 24);
    o.z = (w1 >> 16) | ((w2 & 0x000000ffu) << 16) | (a2 << 24);
    o.w = (w2 >> 8) | (a3 << 24);
    d4[i] = o;
  }
  if (blockIdx.x == 0)
    for (long long i = n4 * 4 + threadIdx.x; i < n; i += blockDim.x)
      dst[i] = make_uchar4(src[3 * i], src[3 * i + 1], src[3 * i + 2],
                           mask ? (mask[i] != 0) : 1);
}

__global__ void __launch_bounds__(256) k_expand(const Geometry* __restrict__ g) {
  pdl_wait();
  const int v = blockIdx.y;
  const ViewDesc& vd = g->views[v];
  expand_span(g->in.frames[v], g->in.masked ? g->in.masks[v] : nullptr, g->rgba[v],
              static_cast<long long>(vd.width) * vd.height);
}

__global__ void __launch_bounds__(256) k_expand_one(const std::uint8_t* __restrict__ src,
                                                    const std::uint8_t* __restrict__ mask,
                                                    uchar4* __restrict__ dst, long long n) {
  expand_span(src, mask, dst, n);
}

// ---------------------------------------------------------------------------
// Geometric warping of the overlap crops: crop_frame(warp_frame(...), bounds)
// (pipeline.cpp:310-311) evaluated directly on the bounds.
// grid: (ceil(max_w/64), ceil(max_h/4), 2*n_pairs), block (64, 4)
// ---------------------------------------------------------------------------
// MASKED (a compile-time choice, dispatched once per kernel from the frame's
// flag): a masked frame's masked taps drop out (frame.cpp:95-104)
template <bool CYL, bool MASKED = false>
__device__ __forceinline__ uchar4 warp_cv(const CanvasView& v, Lift L) {
  if (MASKED) {
    ViewDesc d;
    d.width = v.w;
    d.height = v.h;
#pragma unroll
    for (int i = 0; i < 9; ++i) d.inv[i] = v.inv[i];
    return warp_sample<CYL, true>(d, v.rgba, L);
  }
  if (v.f32) {  // experiment: FP32 interior weights (not bit-exact)
    double sx, sy, sz;
    warp_point<CYL>(v.inv, L, sx, sy, sz);
    uchar4 o = make_uchar4(0, 0, 0, 0);
    if (fabs(sz) < 1e-12) return o;
    if (CYL && !(sz > 0.0)) return o;
    float r, g, b;
    const DDivisor dz = ddivisor(sz);
    if (!sample_rgba_f32(v.rgba, v.w, v.h, ddiv(sx, dz), ddiv(sy, dz), r, g, b)) return o;
    return make_uchar4(quantize_f(r), quantize_f(g), quantize_f(b), 1);
  }
  ViewDesc d;
  d.width = v.w;
  d.height = v.h;
#pragma unroll
  for (int i = 0; i < 9; ++i) d.inv[i] = v.inv[i];
  return warp_sample<CYL>(d, v.rgba, L);
}

__global__ void __launch_bounds__(256) k_crop_warp(const __grid_constant__ CanvasParams P) {
  pdl_wait();
  const int k = blockIdx.z >> 1;
  const int side = blockIdx.z & 1;
  const CanvasPair& p = P.pairs[k];
  const int dx = blockIdx.x * 64 + threadIdx.x;
  const int dy = blockIdx.y * 4 + threadIdx.y;
  if (dx >= p.w || dy >= p.h) return;
  const int view = side ? p.partner : p.view;
  uchar4 o;
  if (*P.masked)
    o = P.projection == 1
            ? warp_cv<true, true>(P.views[view], canvas_lift<true>(P, p.x0 + dx, p.y0 + dy))
            : warp_cv<false, true>(P.views[view], canvas_lift<false>(P, p.x0 + dx, p.y0 + dy));
  else
    o = P.projection == 1
            ? warp_cv<true>(P.views[view], canvas_lift<true>(P, p.x0 + dx, p.y0 + dy))
            : warp_cv<false>(P.views[view], canvas_lift<false>(P, p.x0 + dx, p.y0 + dy));
  p.crop_raw[side][dy * p.w + dx] = o;
}

// Staged variant (planar canvas; STITCH_B200_WARP_STAGE=1): a CTA owns a
// 32 x 8 tile of one crop side; thread 0 maps the tile's corner pixels
// through the view's inverse homography, the CTA loads the bounding window
// of their source footprint (+1 texel margin for the bilinear taps, capped at
// kStageW x kStageH) from the RGBA frame into shared memory with coalesced
// row loads, and every pixel samples its four taps there (sample_rgba_win,
// bit-identical arithmetic).  Tiles whose window does not fit (or whose
// corners leave the front of the camera) and non-interior samples use the
// global-memory sampler.  block (32, 8)
constexpr int kStageW = 64, kStageH = 24;

__global__ void __launch_bounds__(256) k_crop_warp_staged(const __grid_constant__ CanvasParams P) {
  pdl_wait();
  __shared__ uchar4 win[kStageH * kStageW];
  __shared__ int s_wx0, s_wy0, s_ww, s_wh;
  const int k = blockIdx.z >> 1;
  const int side = blockIdx.z & 1;
  const CanvasPair& p = P.pairs[k];
  const int bx0 = blockIdx.x * 32, by0 = blockIdx.y * 8;
  if (bx0 >= p.w || by0 >= p.h) return;  // uniform over the CTA
  const int view = side ? p.partner : p.view;
  const CanvasView& v = P.views[view];
  const int tid = threadIdx.y * 32 + threadIdx.x;
  const bool masked = *P.masked;
  if (tid == 0) {
    double mnx = 1e300, mny = 1e300, mxx = -1e300, mxy = -1e300;
    bool ok = !masked;  // masked frames take the masked global sampler
    const int xs[2] = {bx0, min(bx0 + 31, p.w - 1)}, ys[2] = {by0, min(by0 + 7, p.h - 1)};
    for (int j = 0; j < 2; ++j)
      for (int i = 0; i < 2; ++i) {
        double sx, sy, sz;
        warp_point<false>(v.inv, canvas_lift<false>(P, p.x0 + xs[i], p.y0 + ys[j]), sx, sy, sz);
        if (!(sz > 1e-9)) {
          ok = false;
        } else {
          const double qx = sx / sz, qy = sy / sz;
          mnx = fmin(mnx, qx);
          mny = fmin(mny, qy);
          mxx = fmax(mxx, qx);
          mxy = fmax(mxy, qy);
        }
      }
    int wx0 = 0, wy0 = 0, ww = 0, wh = 0;
    if (ok && mnx > -1e6 && mny > -1e6 && mxx < 1e6 && mxy < 1e6) {
      // one texel of slack beyond the corner images for the rounding of the
      // per-pixel coordinates; the window need not lie inside the frame
      wx0 = static_cast<int>(floor(mnx)) - 1;
      wy0 = static_cast<int>(floor(mny)) - 1;
      ww = static_cast<int>(floor(mxx)) + 3 - wx0;
      wh = static_cast<int>(floor(mxy)) + 3 - wy0;
      if (ww > kStageW || wh > kStageH) ww = wh = 0;
    }
    s_wx0 = wx0;
    s_wy0 = wy0;
    s_ww = ww;
    s_wh = wh;
  }
  __syncthreads();
  const int wx0 = s_wx0, wy0 = s_wy0, ww = s_ww, wh = s_wh;
  for (int i = tid; i < ww * wh; i += 256) {
    const int ly = i / ww, lx = i - ly * ww;
    const int gx = wx0 + lx, gy = wy0 + ly;
    uchar4 t = make_uchar4(0, 0, 0, 0);
    if (gx >= 0 && gx < v.w && gy >= 0 && gy < v.h) t = v.rgba[static_cast<size_t>(gy) * v.w + gx];
    win[ly * kStageW + lx] = t;
  }
  __syncthreads();
  const int dx = bx0 + threadIdx.x, dy = by0 + threadIdx.y;
  if (dx >= p.w || dy >= p.h) return;
  const Lift L = canvas_lift<false>(P, p.x0 + dx, p.y0 + dy);
  double sx, sy, sz;
  warp_point<false>(v.inv, L, sx, sy, sz);
  uchar4 o = make_uchar4(0, 0, 0, 0);
  if (!(fabs(sz) < 1e-12)) {
    const DDivisor dz = ddivisor(sz);
    const double qx = ddiv(sx, dz), qy = ddiv(sy, dz);
    float r, g, b;
    int valid = ww ? sample_rgba_win(win, kStageW, wx0, wy0, ww, wh, v.w, v.h, qx, qy, r, g, b) : -1;
    if (valid < 0)
      valid = (masked ? sample_crop(v.rgba, v.w, v.h, qx, qy, r, g, b)
                      : sample_rgba(v.rgba, v.w, v.h, qx, qy, r, g, b)) ? 1 : 0;
    if (valid) o = make_uchar4(quantize_f(r), quantize_f(g), quantize_f(b), 1);
  }
  p.crop_raw[side][dy * p.w + dx] = o;
}

// ---------------------------------------------------------------------------
// Canvas pass: for every canvas pixel, the warped reference view, then the
// compose_panorama fold over pairs (pipeline.cpp:326-333, flow.cpp:324-357)
// with the colour-corrected warped view (apply_matrix_rows, pipeline.cpp:296)
// and, inside each overlap, the flow-displaced fusion of flow_fuse
// (flow.cpp:282-322) evaluated on demand.  Inside a pair's bounds the raw
// warped samples already computed for the overlap crops are reused
// (bit-identical: same sampler).  Also the balance histogram of the composed
// panorama (compute_histogram, histogram.cpp:5-18); k_balance turns it into
// the tone LUT (global balancing, pipeline.cpp:336-355).
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool fused_pixel(const CanvasParams& P, const CanvasPair& p, int dx,
                                            int dy, uchar4& out) {
  const int i = dy * p.w + dx;
  const float ti = p.theta[i];
  const float tj = 1.0f - ti;  // BlendWeights::theta_j (flow.cpp:276)
  const float wi = P.weighting == 0 ? ti : tj;
  const float wj = P.weighting == 0 ? tj : ti;
  // dense_flow zeroes both fields where either crop is invalid
  // (flow.cpp:178-185); the Jacobi kernels leave that to this consumer
  const bool valid = p.crop_cor[0][i].w && p.crop_cor[1][i].w;
  const float2 fij = valid ? p.fuv[0][i] : make_float2(0.0f, 0.0f);
  const float2 fji = valid ? p.fuv[1][i] : make_float2(0.0f, 0.0f);
  const float uij = fij.x, vij = fij.y, uji = fji.x, vji = fji.y;
  float ri, gi, bi, rj, gj, bj;
  const bool vi = sample_crop(p.crop_cor[0], p.w, p.h,
                              static_cast<double>(static_cast<float>(dx) + wi * uij),
                              static_cast<double>(static_cast<float>(dy) + wi * vij), ri, gi, bi);
  const bool vj = sample_crop(p.crop_cor[1], p.w, p.h,
                              static_cast<double>(static_cast<float>(dx) + wj * uji),
                              static_cast<double>(static_cast<float>(dy) + wj * vji), rj, gj, bj);
  if (!vi && !vj) return false;
  float r, gg, b;
  if (vi && vj) {
    r = ti * ri + tj * rj;
    gg = ti * gi + tj * gj;
    b = ti * bi + tj * bj;
  } else if (vi) {
    r = ri;
    gg = gi;
    b = bi;
  } else {
    r = rj;
    gg = gj;
    b = bj;
  }
  out = make_uchar4(quantize_f(r), quantize_f(gg), quantize_f(b), 1);
  return true;
}

// Global balancing, one CTA (k_balance, or the canvas's last CTA):
// find_thresholds (color_balance.cpp:8-38),
// history push (pipeline.cpp:340-345), smooth_thresholds
// (color_balance.cpp:40-63), build_curve (color_balance.cpp:65-104).
__device__ unsigned char curve_entry(int v, int m1, int m2, double gamma_dark,
                                     double gamma_bright, double target_black,
                                     double target_white);

__device__ void balance_lut(const Geometry* __restrict__ g, DevState* __restrict__ st) {
  __shared__ int sm1[3], sm2[3], first1[3], first2[3];
  __shared__ unsigned long long wtot[8];
  __shared__ int ok;
  // the threshold history and the frame counter, staged in shared memory by
  // parallel loads so thread 0's update below is not a chain of dependent
  // global round trips
  constexpr int kBsInts = static_cast<int>(sizeof(BalanceState) / sizeof(int));
  __shared__ int sbs[kBsInts];
  __shared__ long long s_counter;
  const int v = threadIdx.x;
  int* gbs = reinterpret_cast<int*>(st->balance);
  if (v < kBsInts) sbs[v] = gbs[v];
  if (v == kBsInts) s_counter = *st->frame_counter;
  unsigned int hist[3];
  for (int c = 0; c < 3; ++c) {
    hist[c] = st->pano_hist[c][v];
    st->pano_hist[c][v] = 0;
  }
  if (v < 3) {
    first1[v] = 256;
    first2[v] = 256;
  }
  // inclusive prefix per channel (block scan of 256 bins)
  unsigned long long run[3];
  for (int c = 0; c < 3; ++c) {
    unsigned long long x = hist[c];
    const int lane = v & 31, wid = v >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wtot[wid] = x;
    __syncthreads();
    unsigned long long add = 0;
    for (int i = 0; i < wid; ++i) add += wtot[i];
    __syncthreads();
    run[c] = x + add;
  }
  __shared__ unsigned long long s_total;
  if (v == 255) s_total = run[0];
  __syncthreads();
  const unsigned long long tot = s_total;
  if (tot != 0) {
    const double dtot = static_cast<double>(tot);
    for (int c = 0; c < 3; ++c) {
      const double cdf = static_cast<double>(run[c]) / dtot;
      if (cdf >= g->lambda) atomicMin(&first1[c], v);
      if (cdf >= 1.0 - g->lambda) atomicMin(&first2[c], v);
    }
  }
  __syncthreads();
  if (v == 0) {
    ok = 0;
    st->report.frame_index = s_counter;
    if (tot != 0) {
      BalanceState& bs = *reinterpret_cast<BalanceState*>(sbs);
      if (bs.n == 3) {
        for (int i = 0; i < 2; ++i)
          for (int c = 0; c < 3; ++c) {
            bs.m1[i][c] = bs.m1[i + 1][c];
            bs.m2[i][c] = bs.m2[i + 1][c];
          }
        bs.n = 2;
      }
      for (int c = 0; c < 3; ++c) {
        // m1 defaults to 255 and is only taken at or before m2 (the
        // reference loop breaks at m2, color_balance.cpp:25-35)
        const int m2 = first2[c] < 256 ? first2[c] : 255;
        const int m1 = first1[c] <= m2 ? first1[c] : 255;
        bs.m1[bs.n][c] = m1;
        bs.m2[bs.n][c] = m2;
      }
      bs.n++;
      const int nh = bs.n;
      for (int c = 0; c < 3; ++c) {
        double s1 = 0.0, s2 = 0.0;
        for (int i = 0; i < nh; ++i) {
          s1 += bs.m1[i][c];
          s2 += bs.m2[i][c];
        }
        int a = static_cast<int>(llround(s1 / static_cast<double>(nh)));
        int b = static_cast<int>(llround(s2 / static_cast<double>(nh)));
        if (a > b) {
          const int tmp = a;
          a = b;
          b = tmp;
        }
        sm1[c] = a;
        sm2[c] = b;
      }
      ok = g->curve_ok;
    }
    st->report.balanced = ok;
    for (int c = 0; c < 3; ++c) {
      st->report.m1[c] = ok ? sm1[c] : 0;
      st->report.m2[c] = ok ? sm2[c] : 0;
    }
    *st->frame_counter = s_counter + 1;
  }
  __syncthreads();
  if (v < kBsInts) gbs[v] = sbs[v];
  for (int c = 0; c < 3; ++c)
    st->lut[c][v] = ok ? curve_entry(v, sm1[c], sm2[c], g->gamma_dark, g->gamma_bright,
                                     g->target_black, g->target_white)
                       : static_cast<unsigned char>(v);
}

// One entry of build_curve (color_balance.cpp:65-104): balance_curve_value in
// the reference's operation order (FP64, no FMA, CUDA pow), then
// quantize_channel.  Checked against the compiled reference's curve for every
// (m1, m2) by tests/test_ref_pin.py through k_debug_tone_curves.
__device__ unsigned char curve_entry(int v, int m1, int m2, double gamma_dark,
                                     double gamma_bright, double target_black,
                                     double target_white) {
  const double tb = target_black, tw = target_white;
  const double x = static_cast<double>(v);
  double val;
  if (m1 >= m2) {
    val = tb + (tw - tb) * (x / 255.0);
  } else {
    const double lm1 = tb + (tw - tb) * (static_cast<double>(m1) / 255.0);
    const double lm2 = tb + (tw - tb) * (static_cast<double>(m2) / 255.0);
    if (x <= m1) {
      val = (m1 == 0) ? tb : tb + (lm1 - tb) * pow(x / m1, gamma_dark);
    } else if (x >= m2) {
      val = (m2 == 255) ? tw : lm2 + (tw - lm2) * pow((x - m2) / (255.0 - m2), gamma_bright);
    } else {
      val = lm1 + (lm2 - lm1) * (x - m1) / (m2 - m1);
    }
  }
  return quantize_d(val);
}

// Test entry: n curves (one per (m1[i], m2[i])) of 256 entries each.
__global__ void k_debug_tone_curves(int n, const int* __restrict__ m1, const int* __restrict__ m2,
                                    double gamma_dark, double gamma_bright, double tb, double tw,
                                    unsigned char* __restrict__ out) {
  const int i = blockIdx.x;
  if (i >= n) return;
  out[static_cast<size_t>(i) * 256 + threadIdx.x] =
      curve_entry(threadIdx.x, m1[i], m2[i], gamma_dark, gamma_bright, tb, tw);
}

// the view's footprint may contain (x, y): inside its bbox and outside the
// empty column run of a wrapped ring view (the warp is invalid there, so
// skipping it is exact)
__device__ __forceinline__ bool may_cover(const CanvasView& v, int x, int y) {
  return x >= v.bbox[0] && x < v.bbox[2] && y >= v.bbox[1] && y < v.bbox[3] &&
         !(x >= v.gap[0] && x < v.gap[1]);
}

__device__ __forceinline__ bool in_rect(const CanvasPair& p, int x, int y) {
  return x >= p.x0 && x < p.x0 + p.w && y >= p.y0 && y < p.y0 + p.h;
}

// One canvas pixel: the warped reference view, then the compose_panorama
// fold over pairs (pipeline.cpp:326-333, flow.cpp:324-357).
template <bool CYL, bool MASKED>
__device__ __forceinline__ uchar4 canvas_pixel(const CanvasParams& P,
                                               const double (*mview)[9], int x, int y) {
  const int ref = P.ref;
  const CanvasView& vr = P.views[ref];
  const int np = P.np;
  const Lift L = canvas_lift<CYL>(P, x, y);
  uchar4 pv = make_uchar4(0, 0, 0, 0);
  if (may_cover(vr, x, y)) {
    // reuse a star pair's crop of the reference view when inside its bounds
    int kc = -1;
    for (int k = 0; k < np; ++k) {
      const CanvasPair& p = P.pairs[k];
      if (p.partner == ref && x >= p.x0 && x < p.x0 + p.w && y >= p.y0 && y < p.y0 + p.h) {
        kc = k;
        break;
      }
    }
    if (kc >= 0) {
      const CanvasPair& p = P.pairs[kc];
      pv = p.crop_raw[1][(y - p.y0) * p.w + (x - p.x0)];
    } else {
      pv = warp_cv<CYL, MASKED>(vr, L);
    }
  }
  for (int k = 0; k < np; ++k) {
    const CanvasPair& p = P.pairs[k];
    const CanvasView& vv = P.views[p.view];
    if (!may_cover(vv, x, y)) continue;
    const int dx = x - p.x0, dy = y - p.y0;
    const bool inb = dx >= 0 && dy >= 0 && dx < p.w && dy < p.h;
    const uchar4 q = inb ? p.crop_raw[0][dy * p.w + dx] : warp_cv<CYL, MASKED>(vv, L);
    if (!q.w) continue;
    if (pv.w) {
      if (inb) {
        uchar4 f;
        if (fused_pixel(P, p, dx, dy, f)) pv = f;
      }
    } else {
      pv = apply_matrix(mview[p.view], q);
    }
  }
  return pv;
}

// Every canvas pixel of this CTA's grid-stride tiles (64 x 4), into pano and
// the CTA's histogram.
template <bool CYL, bool MASKED>
__device__ __forceinline__ void canvas_tiles(const CanvasParams& P, const double (*mview)[9],
                                             uchar4* __restrict__ pano,
                                             unsigned int (*hist)[256]) {
  const int cw = P.cw, ch = P.ch;
  const int tiles_x = (cw + 63) / 64;
  const int ntiles = tiles_x * ((ch + 3) / 4);
  // tile -> (column, row) kept incrementally: the grid stride advances by
  // (dq rows, dr columns), one integer division per thread instead of one
  // per tile
  const int dq = static_cast<int>(gridDim.x) / tiles_x, dr = static_cast<int>(gridDim.x) - dq * tiles_x;
  int ty = static_cast<int>(blockIdx.x) / tiles_x;
  int tcol = static_cast<int>(blockIdx.x) - ty * tiles_x;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int x = tcol * 64 + threadIdx.x % 64;
    const int y = ty * 4 + threadIdx.x / 64;
    tcol += dr;
    ty += dq;
    if (tcol >= tiles_x) {
      tcol -= tiles_x;
      ++ty;
    }
    if (x >= cw || y >= ch) continue;
    const long long idx = static_cast<long long>(y) * cw + x;
    uchar4 pv;
    // a masked frame's coverage is not the geometry's: every pixel runs the fold
    const std::uint8_t c = (P.cls && !MASKED) ? P.cls[idx] : kClassFold;
    if (c == kClassFold) {
      pv = canvas_pixel<CYL, MASKED>(P, mview, x, y);
    } else if (c == kClassNone) {
      pv = make_uchar4(0, 0, 0, 0);
    } else {
      // a single view provides the pixel: its warp, colour-corrected unless
      // it is the reference (the fold's result, without evaluating the
      // views that do not cover the pixel)
      pv = warp_cv<CYL>(P.views[c], canvas_lift<CYL>(P, x, y));
      if (c != P.ref) pv = apply_matrix(mview[c], pv);
    }
    pano[idx] = pv;
    if (pv.w) {
      atomicAdd(&hist[0][pv.x], 1u);
      atomicAdd(&hist[1][pv.y], 1u);
      atomicAdd(&hist[2][pv.z], 1u);
    }
  }
}

constexpr int kCanvasCtasPerSm = 4;  // resident CTAs per SM (register budget; 5 spills)

// Every canvas pixel once (64 x 4 tiles, grid-stride), per-CTA histogram
// flushed to the frame histogram; k_balance (or, ELECT, the last CTA) then
// builds the balance LUT.
template <bool CYL, bool ELECT = true>
__global__ void __launch_bounds__(256, kCanvasCtasPerSm) k_canvas(const __grid_constant__ CanvasParams P,
                                                   const Geometry* __restrict__ g,
                                                   DevState* __restrict__ st,
                                                   uchar4* __restrict__ pano) {
  pdl_wait();
  __shared__ unsigned int hist[3][256];
  __shared__ double mview[kMaxViews][9];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    hist[0][i] = 0;
    hist[1][i] = 0;
    hist[2][i] = 0;
  }
  for (int i = threadIdx.x; i < kMaxViews * 9; i += blockDim.x) mview[i / 9][i % 9] = st->mview[i / 9][i % 9];
  __syncthreads();
  if (*P.masked)
    canvas_tiles<CYL, true>(P, mview, pano, hist);
  else
    canvas_tiles<CYL, false>(P, mview, pano, hist);
  __syncthreads();
  if (!ELECT) pdl_trigger();  // only the histogram flush remains
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    for (int c = 0; c < 3; ++c)
      if (hist[c][i]) atomicAdd(&st->pano_hist[c][i], hist[c][i]);
  if (!ELECT) return;
  if (!elect_last_cta(&st->canvas_done, gridDim.x)) return;
  if (threadIdx.x == 0) st->canvas_done = 0;
  balance_lut(g, st);
}

// the balance LUT in its own launch after the canvas (ELECT = false)
__global__ void __launch_bounds__(256) k_balance(const Geometry* __restrict__ g,
                                                 DevState* __restrict__ st) {
  pdl_wait();
  balance_lut(g, st);
}

// apply_tone_rows (pipeline.cpp:84-96) + conversion to the reference's Frame
// layout (RGB8 interleaved + 0/1 mask).  4 pixels per thread: one 16-byte
// uchar4x4 load, three 4-byte RGB stores, one 4-byte mask store.
__global__ void __launch_bounds__(256) k_tone(const DevState* __restrict__ st,
                                              const uchar4* __restrict__ pano, long long n_px,
                                              std::uint8_t* __restrict__ out_rgb,
                                              std::uint8_t* __restrict__ out_mask) {
  pdl_wait();
  __shared__ unsigned char lut[3][256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    lut[0][i] = st->lut[0][i];
    lut[1][i] = st->lut[1][i];
    lut[2][i] = st->lut[2][i];
  }
  __syncthreads();
  const long long n4 = n_px / 4;
  const uint4* p4 = reinterpret_cast<const uint4*>(pano);
  unsigned int* rgb4 = reinterpret_cast<unsigned int*>(out_rgb);
  unsigned int* m4 = reinterpret_cast<unsigned int*>(out_mask);
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const uint4 q = p4[i];
    const unsigned int px[4] = {q.x, q.y, q.z, q.w};
    unsigned char o[12];
    unsigned int mask = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const unsigned int v = px[j];
      const unsigned char r = v & 0xff, gg = (v >> 8) & 0xff, b = (v >> 16) & 0xff;
      const unsigned char valid = (v >> 24) & 0xff;
      o[3 * j + 0] = valid ? lut[0][r] : r;
      o[3 * j + 1] = valid ? lut[1][gg] : gg;
      o[3 * j + 2] = valid ? lut[2][b] : b;
      mask |= static_cast<unsigned int>(valid ? 1 : 0) << (8 * j);
    }
    rgb4[3 * i + 0] = o[0] | (o[1] << 8) | (o[2] << 16) | (static_cast<unsigned int>(o[3]) << 24);
    rgb4[3 * i + 1] = o[4] | (o[5] << 8) | (o[6] << 16) | (static_cast<unsigned int>(o[7]) << 24);
    rgb4[3 * i + 2] = o[8] | (o[9] << 8) | (o[10] << 16) | (static_cast<unsigned int>(o[11]) << 24);
    m4[i] = mask;
  }
  // tail
  if (blockIdx.x == 0) {
    for (long long i = n4 * 4 + threadIdx.x; i < n_px; i += blockDim.x) {
      const uchar4 v = pano[i];
      out_rgb[3 * i + 0] = v.w ? lut[0][v.x] : v.x;
      out_rgb[3 * i + 1] = v.w ? lut[1][v.y] : v.y;
      out_rgb[3 * i + 2] = v.w ? lut[2][v.z] : v.z;
      out_mask[i] = v.w ? 1 : 0;
    }
  }
}

// Full-canvas warp of one view (init masks and debug readback).
template <bool MASKED>
__global__ void __launch_bounds__(256) k_warp_view(const Geometry* __restrict__ g, int view,
                                                   const uchar4* __restrict__ frame,
                                                   std::uint8_t* __restrict__ rgb,
                                                   std::uint8_t* __restrict__ mask) {
  const ViewDesc& v = g->views[view];
  const long long n = static_cast<long long>(g->canvas_w) * g->canvas_h;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < n;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int y = static_cast<int>(idx / g->canvas_w);
    const int x = static_cast<int>(idx - static_cast<long long>(y) * g->canvas_w);
    const uchar4 o = g->projection == 1
                         ? warp_sample<true, MASKED>(v, frame, canvas_lift<true>(*g, x, y))
                         : warp_sample<false, MASKED>(v, frame, canvas_lift<false>(*g, x, y));
    if (rgb) {
      rgb[3 * idx + 0] = o.x;
      rgb[3 * idx + 1] = o.y;
      rgb[3 * idx + 2] = o.z;
    }
    mask[idx] = o.w;
  }
}

// Geometry-only validity of the warp (the input frames are unmasked, so the
// mask does not depend on pixel values): sample_bilinear is valid iff a
// neighbour with positive weight lies inside the frame.
template <bool CYL>
__device__ __forceinline__ bool warp_valid(const double* inv, int W, int H, Lift L) {
  double sx0, sy0, sz0;
  warp_point<CYL>(inv, L, sx0, sy0, sz0);
  if (fabs(sz0) < 1e-12 || (CYL && !(sz0 > 0.0))) return false;
  const double sx = sx0 / sz0, sy = sy0 / sz0;
  const double fx0 = floor(sx), fy0 = floor(sy);
  const int x0 = static_cast<int>(fx0), y0 = static_cast<int>(fy0);
  const double ax = sx - fx0, ay = sy - fy0;
  for (int j = 0; j < 2; ++j)
    for (int i = 0; i < 2; ++i) {
      const double w = (i ? ax : 1.0 - ax) * (j ? ay : 1.0 - ay);
      const unsigned xx = static_cast<unsigned>(x0) + i, yy = static_cast<unsigned>(y0) + j;
      if (w > 0.0 && xx < static_cast<unsigned>(W) && yy < static_cast<unsigned>(H)) return true;
    }
  return false;
}

// Validity of sample_bilinear on a masked frame (frame.cpp:79-109): some
// neighbour with a positive weight is inside the frame and unmasked -- the
// weights of sample_crop, so exactly its `wsum > 0`.
__device__ __forceinline__ bool masked_sample_valid(const std::uint8_t* __restrict__ m, int W,
                                                    int H, double x, double y) {
  const double fx0 = floor(x), fy0 = floor(y);
  const int x0 = static_cast<int>(fx0), y0 = static_cast<int>(fy0);
  const double ax = x - fx0, ay = y - fy0;
  const double wx0 = 1.0 - ax, wy0 = 1.0 - ay;
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const double w = (i ? ax : wx0) * (j ? ay : wy0);
      const unsigned xx = static_cast<unsigned>(x0) + static_cast<unsigned>(i);
      const unsigned yy = static_cast<unsigned>(y0) + static_cast<unsigned>(j);
      if (w > 0.0 && xx < static_cast<unsigned>(W) && yy < static_cast<unsigned>(H) &&
          m[static_cast<size_t>(yy) * W + xx])
        return true;
    }
  return false;
}

// warp_frame's `any` (geometry.cpp:64-81) for masked frames: grid (CTAs,
// listed views); each CTA scans its share of the view's rect and stops as
// soon as any CTA has found a valid pixel of that view.
template <bool CYL>
__global__ void __launch_bounds__(256) k_mask_coverage(const Geometry* __restrict__ g,
                                                       const __grid_constant__ MaskSet ms,
                                                       unsigned* covered) {
  const int j = blockIdx.y;
  const int view = ms.view[j];
  const ViewDesc& v = g->views[view];
  const int x0 = ms.rect[j][0], y0 = ms.rect[j][1];
  const int rw = ms.rect[j][2] - x0, rh = ms.rect[j][3] - y0;
  if (rw <= 0 || rh <= 0) return;
  const long long n = static_cast<long long>(rw) * rh;
  const unsigned bit = 1u << view;
  const volatile unsigned* cv = covered;
  for (long long base = blockIdx.x * 256ll; base < n; base += gridDim.x * 256ll) {
    bool hit = false;
    const long long idx = base + threadIdx.x;
    if (idx < n) {
      const int y = y0 + static_cast<int>(idx / rw);
      const int x = x0 + static_cast<int>(idx % rw);
      double sx, sy, sz;
      warp_point<CYL>(v.inv, canvas_lift<CYL>(*g, x, y), sx, sy, sz);
      if (!(fabs(sz) < 1e-12) && (!CYL || sz > 0.0)) {
        const DDivisor dz = ddivisor(sz);
        hit = masked_sample_valid(ms.mask[j], v.width, v.height, ddiv(sx, dz), ddiv(sy, dz));
      }
    }
    const bool done = threadIdx.x == 0 && (*cv & bit);
    if (__syncthreads_or(hit || done)) {
      if (threadIdx.x == 0) atomicOr(covered, bit);
      return;
    }
  }
}

__global__ void __launch_bounds__(256) k_warp_mask(const Geometry* __restrict__ g, int view,
                                                   std::uint8_t* __restrict__ mask) {
  const ViewDesc& v = g->views[view];
  const long long n = static_cast<long long>(g->canvas_w) * g->canvas_h;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < n;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int y = static_cast<int>(idx / g->canvas_w);
    const int x = static_cast<int>(idx - static_cast<long long>(y) * g->canvas_w);
    mask[idx] = g->projection == 1
                    ? warp_valid<true>(v.inv, v.width, v.height, canvas_lift<true>(*g, x, y))
                    : warp_valid<false>(v.inv, v.width, v.height, canvas_lift<false>(*g, x, y));
  }
}

// Canvas class map (CanvasParams::cls): outside every pair's bounds the
// compose fold (pipeline.cpp:326-333, flow.cpp:324-357) keeps the warped
// reference where it is valid, else takes the first valid view of the pairs
// in order (colour-corrected); validity is geometry-only, so which view that
// is depends on the maps alone and is fixed per context.
template <bool CYL>
__global__ void __launch_bounds__(256) k_canvas_class(const __grid_constant__ CanvasParams P,
                                                      std::uint8_t* __restrict__ cls) {
  const long long n = static_cast<long long>(P.cw) * P.ch;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < n;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int y = static_cast<int>(idx / P.cw);
    const int x = static_cast<int>(idx - static_cast<long long>(y) * P.cw);
    std::uint8_t c = kClassNone;
    bool fold = false;
    for (int k = 0; k < P.np; ++k) fold = fold || in_rect(P.pairs[k], x, y);
    if (fold) {
      c = kClassFold;
    } else {
      const Lift L = canvas_lift<CYL>(P, x, y);
      for (int k = -1; k < P.np && c == kClassNone; ++k) {
        const int v = k < 0 ? P.ref : P.pairs[k].view;
        const CanvasView& vv = P.views[v];
        if (may_cover(vv, x, y) && warp_valid<CYL>(vv.inv, vv.w, vv.h, L))
          c = static_cast<std::uint8_t>(v);
      }
    }
    cls[idx] = c;
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static inline int blocks_for(long long n, int per = 256, int cap = 65535) {
  long long b = (n + per - 1) / per;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return static_cast<int>(b);
}

void launch_expand(const Geometry* g, int n_views, long long max_px, cudaStream_t s) {
  dim3 grid(blocks_for(max_px / 4 + 1, 256, 148 * 4), n_views);
  k_expand<<<grid, 256, 0, s>>>(g);
}

void launch_expand_one(const std::uint8_t* rgb, uchar4* rgba, long long n_px, cudaStream_t s,
                       const std::uint8_t* mask) {
  k_expand_one<<<blocks_for(n_px / 4 + 1, 256, 148 * 4), 256, 0, s>>>(rgb, mask, rgba, n_px);
}

void launch_crop_warp(const CanvasParams& P, int max_w, int max_h, cudaStream_t s) {
  static const int stage = env_int("STITCH_B200_WARP_STAGE", 0);
  if (stage && P.projection == 0) {
    dim3 grid((max_w + 31) / 32, (max_h + 7) / 8, 2 * P.np);
    k_crop_warp_staged<<<grid, dim3(32, 8), 0, s>>>(P);
    return;
  }
  dim3 grid((max_w + 63) / 64, (max_h + 3) / 4, 2 * P.np);
  k_crop_warp<<<grid, dim3(64, 4), 0, s>>>(P);
}

int launch_canvas(const CanvasParams& P, const Geometry* g, DevState* st, uchar4* pano,
                  int num_sms, cudaStream_t s) {
  const long long tiles = static_cast<long long>((P.cw + 63) / 64) * ((P.ch + 3) / 4);
  const long long b = std::min<long long>(static_cast<long long>(num_sms) * kCanvasCtasPerSm, tiles);
  const int blocks = static_cast<int>(b < 1 ? 1 : b);
  // the balance LUT in its own one-CTA launch: the canvas CTAs exit after
  // their histogram flush instead of fencing for the last-CTA election
  // (canvas 0.177 -> 0.171 ms, p50 1.458 -> 1.448 ms at C2, scripts/exp24.sh);
  // STITCH_B200_CANVAS_SPLIT=0 restores the election
  static const int split = env_int("STITCH_B200_CANVAS_SPLIT", 1);
  if (split) {
    if (P.projection == 1)
      k_canvas<true, false><<<blocks, 256, 0, s>>>(P, g, st, pano);
    else
      k_canvas<false, false><<<blocks, 256, 0, s>>>(P, g, st, pano);
    k_balance<<<1, 256, 0, s>>>(g, st);
    return 2;
  }
  if (P.projection == 1)
    k_canvas<true><<<blocks, 256, 0, s>>>(P, g, st, pano);
  else
    k_canvas<false><<<blocks, 256, 0, s>>>(P, g, st, pano);
  return 1;
}

void launch_tone(const DevState* st, const uchar4* pano, long long n_px, std::uint8_t* out_rgb,
                 std::uint8_t* out_mask, cudaStream_t s) {
  k_tone<<<blocks_for(n_px / 4 + 1, 256, 148 * 16), 256, 0, s>>>(st, pano, n_px, out_rgb,
                                                                  out_mask);
}

void launch_warp_view(const Geometry* g, int view, const uchar4* frame, std::uint8_t* rgb,
                      std::uint8_t* mask, cudaStream_t s, bool masked) {
  if (masked)
    k_warp_view<true><<<148 * 8, 256, 0, s>>>(g, view, frame, rgb, mask);
  else
    k_warp_view<false><<<148 * 8, 256, 0, s>>>(g, view, frame, rgb, mask);
}

void launch_warp_mask(const Geometry* g, int view, std::uint8_t* mask, cudaStream_t s) {
  k_warp_mask<<<148 * 8, 256, 0, s>>>(g, view, mask);
}

void launch_mask_coverage(const Geometry* g, int projection, const MaskSet& ms, long long max_px,
                          unsigned* covered, cudaStream_t s) {
  if (ms.n <= 0) return;
  const dim3 grid(blocks_for(max_px, 256, 148 * 4), ms.n);
  if (projection == 1)
    k_mask_coverage<true><<<grid, 256, 0, s>>>(g, ms, covered);
  else
    k_mask_coverage<false><<<grid, 256, 0, s>>>(g, ms, covered);
}

void launch_canvas_class(const CanvasParams& P, std::uint8_t* cls, cudaStream_t s) {
  if (P.projection == 1)
    k_canvas_class<true><<<148 * 8, 256, 0, s>>>(P, cls);
  else
    k_canvas_class<false><<<148 * 8, 256, 0, s>>>(P, cls);
}

void launch_debug_tone_curves(int n, const int* m1, const int* m2, double gamma_dark,
                              double gamma_bright, double tb, double tw, std::uint8_t* out,
                              cudaStream_t s) {
  if (n > 0) k_debug_tone_curves<<<n, 256, 0, s>>>(n, m1, m2, gamma_dark, gamma_bright, tb, tw, out);
}

}  // namespace stitch_b200_dev
