// kernels.cu -- sm_100a kernels of the per-frame stitching path
// (process_frame, /root/reference/proj/src/pipeline.cpp:259-360).
//
// Stage -> kernel map:
//   geometric warping (pipeline.cpp:270-277)    k_crop_warp (overlap crops),
//                                               fused into k_canvas elsewhere
//   3D-M colour transfer (pipeline.cpp:279-300) k_pair_stats -> k_pair_solve
//   local warping / flow (pipeline.cpp:302-322) k_flow_prepare, k_pyr_down,
//                                               k_upsample, k_hs_iter
//   blending (pipeline.cpp:324-334)             k_canvas (warp + M + fuse +
//                                               compose + histogram)
//   global balancing (pipeline.cpp:336-355)     k_balance -> k_tone
#include <cuda_runtime.h>

#include "device_math.cuh"
#include "kernels.cuh"

namespace stitch_b200_dev {

// ---------------------------------------------------------------------------
// Geometric warping of the overlap crops: crop_frame(warp_frame(...), bounds)
// (pipeline.cpp:310-311) evaluated directly on the bounds.
// grid: (x blocks, 2*n_pairs)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_crop_warp(const Geometry* __restrict__ g) {
  const int k = blockIdx.y >> 1;
  const int side = blockIdx.y & 1;
  const PairDesc& p = g->pairs[k];
  const int n = p.w * p.h;
  const int view = side ? p.partner : p.view;
  const ViewDesc& v = g->views[view];
  const std::uint8_t* frame = g->frames[view];
  uchar4* out = p.crop_raw[side];
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += gridDim.x * blockDim.x) {
    const int dy = idx / p.w;
    const int dx = idx - dy * p.w;
    const double X = static_cast<double>(p.x0 + dx) + g->offx;
    const double Y = static_cast<double>(p.y0 + dy) + g->offy;
    out[idx] = warp_sample(v, frame, X, Y);
  }
}

// ---------------------------------------------------------------------------
// transfer_step's single pass over the jointly valid overlap pixels
// (color_transfer.cpp:147-163), reduced to integer tables: source/reference
// histograms and the conditional sums S_{a|b}[v] = sum_{x_b = v} x_a, from
// which X^T X and X^T Y follow exactly (see k_pair_solve).
// grid: (blocks per pair, pairs of this depth)
// ---------------------------------------------------------------------------
__device__ __forceinline__ int sidx(int a, int b) { return a * 2 + (b > a ? b - 1 : b); }

__global__ void __launch_bounds__(256) k_pair_stats(const Geometry* __restrict__ g,
                                                    DevState* __restrict__ st,
                                                    const int* __restrict__ list) {
  __shared__ unsigned int hs[3][256];
  __shared__ unsigned int hr[3][256];
  __shared__ unsigned int ss[6][256];
  __shared__ unsigned int cnt;
  const int k = list[blockIdx.y];
  const PairDesc& p = g->pairs[k];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    for (int c = 0; c < 3; ++c) {
      hs[c][i] = 0;
      hr[c][i] = 0;
    }
    for (int c = 0; c < 6; ++c) ss[c][i] = 0;
  }
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  const bool correct_partner = p.partner != g->reference;
  const double* mp = st->mview[p.partner];
  const int n = p.w * p.h;
  unsigned int local = 0;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += gridDim.x * blockDim.x) {
    const uchar4 a = p.crop_raw[0][idx];
    uchar4 b = p.crop_raw[1][idx];
    if (!a.w || !b.w) continue;
    if (correct_partner) b = apply_matrix(mp, b);
    const unsigned int xa[3] = {a.x, a.y, a.z};
    atomicAdd(&hs[0][a.x], 1u);
    atomicAdd(&hs[1][a.y], 1u);
    atomicAdd(&hs[2][a.z], 1u);
    atomicAdd(&hr[0][b.x], 1u);
    atomicAdd(&hr[1][b.y], 1u);
    atomicAdd(&hr[2][b.z], 1u);
#pragma unroll
    for (int ca = 0; ca < 3; ++ca)
#pragma unroll
      for (int cb = 0; cb < 3; ++cb)
        if (ca != cb) atomicAdd(&ss[sidx(ca, cb)][xa[cb]], xa[ca]);
    ++local;
  }
  atomicAdd(&cnt, local);
  __syncthreads();
  PairStats& out = st->stats[k];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    for (int c = 0; c < 3; ++c) {
      if (hs[c][i]) atomicAdd(&out.hs[c][i], hs[c][i]);
      if (hr[c][i]) atomicAdd(&out.hr[c][i], hr[c][i]);
    }
    for (int c = 0; c < 6; ++c)
      if (ss[c][i]) atomicAdd(&out.s[c][i], static_cast<unsigned long long>(ss[c][i]));
  }
  if (threadIdx.x == 0 && cnt) atomicAdd(&out.n, static_cast<unsigned long long>(cnt));
}

// ---------------------------------------------------------------------------
// Per-pair solve: histogram_specification (color_transfer.cpp:28-55), the
// revised-row moments, TransferWindow push (color_transfer.cpp:16-21),
// solve_color_matrix (color_transfer.cpp:73-99) with the rank guard, and the
// degrade rules of process_frame (pipeline.cpp:282-293).
// One block per pair.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_pair_solve(const Geometry* __restrict__ g,
                                                    DevState* __restrict__ st,
                                                    const int* __restrict__ list) {
  __shared__ unsigned int hs[3][256];
  __shared__ unsigned int hr[3][256];
  __shared__ unsigned long long ss[6][256];
  __shared__ unsigned char lut[3][256];
  __shared__ unsigned long long mom[18];
  const int k = list[blockIdx.x];
  const PairDesc& p = g->pairs[k];
  PairStats& in = st->stats[k];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    for (int c = 0; c < 3; ++c) {
      hs[c][i] = in.hs[c][i];
      hr[c][i] = in.hr[c][i];
    }
    for (int c = 0; c < 6; ++c) ss[c][i] = in.s[c][i];
  }
  const unsigned long long n = in.n;
  __syncthreads();
  // reset the accumulators for the next frame
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    for (int c = 0; c < 3; ++c) {
      in.hs[c][i] = 0;
      in.hr[c][i] = 0;
    }
    for (int c = 0; c < 6; ++c) in.s[c][i] = 0;
  }
  if (threadIdx.x == 0) in.n = 0;

  if (n == 0) {
    // EmptyRegion from transfer_step: identity M, window untouched.
    if (threadIdx.x == 0) {
      for (int i = 0; i < 9; ++i) {
        const double v = (i % 4 == 0) ? 1.0 : 0.0;
        st->mview[p.view][i] = v;
        st->report.m[k][i] = v;
      }
      st->report.rank_deficient[k] = 1;
    }
    return;
  }
  // histogram_specification: one thread per channel.
  if (threadIdx.x < 3) {
    const int c = threadIdx.x;
    unsigned long long cum_ref[256];
    unsigned long long run = 0;
    for (int v = 0; v < 256; ++v) {
      run += hr[c][v];
      cum_ref[v] = run;
    }
    // src and ref share the jointly-valid count n.
    unsigned long long cum_src = 0;
    int u = 0;
    for (int v = 0; v < 256; ++v) {
      cum_src += hs[c][v];
      while (u < 255 && cum_ref[u] * n < cum_src * n) ++u;
      lut[c][v] = static_cast<unsigned char>(u);
    }
  }
  __syncthreads();
  // exact integer moments: X^T X (9) and X^T Y (9)
  if (threadIdx.x < 18) {
    const int which = threadIdx.x / 9;
    const int a = (threadIdx.x % 9) / 3;
    const int b = threadIdx.x % 3;
    unsigned long long acc = 0;
    if (which == 0) {
      if (a == b)
        for (int v = 0; v < 256; ++v) acc += static_cast<unsigned long long>(v) * v * hs[a][v];
      else
        for (int v = 0; v < 256; ++v) acc += static_cast<unsigned long long>(v) * ss[sidx(a, b)][v];
    } else {
      if (a == b)
        for (int v = 0; v < 256; ++v)
          acc += static_cast<unsigned long long>(v) * lut[a][v] * hs[a][v];
      else
        for (int v = 0; v < 256; ++v)
          acc += static_cast<unsigned long long>(lut[b][v]) * ss[sidx(a, b)][v];
    }
    mom[threadIdx.x] = acc;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  PairWindow& w = st->windows[k];
  // push newest first, evict beyond capacity
  int size = w.size < w.capacity ? w.size + 1 : w.capacity;
  for (int i = size - 1; i > 0; --i) w.e[i] = w.e[i - 1];
  for (int i = 0; i < 9; ++i) {
    w.e[0].xtx[i] = mom[i];
    w.e[0].xty[i] = mom[9 + i];
  }
  w.e[0].n = n;
  w.size = size;
  unsigned long long sx[9] = {0}, sy[9] = {0}, total = 0;
  for (int e = 0; e < size; ++e) {
    for (int i = 0; i < 9; ++i) {
      sx[i] += w.e[e].xtx[i];
      sy[i] += w.e[e].xty[i];
    }
    total += w.e[e].n;
  }
  double normal[9], xty[9], m[9], sv[3];
  for (int i = 0; i < 9; ++i) {
    normal[i] = static_cast<double>(sx[i]);
    xty[i] = static_cast<double>(sy[i]);
  }
  sym3_eigen(normal, sv);
  int degraded = 0;
  if (total < 3 || sv[2] < 1e-8 * sv[0]) {
    for (int i = 0; i < 9; ++i) m[i] = (i % 4 == 0) ? 1.0 : 0.0;
    degraded = 1;
  } else {
    ldlt_solve3(normal, xty, m);
  }
  for (int i = 0; i < 9; ++i) {
    st->mview[p.view][i] = m[i];
    st->report.m[k][i] = m[i];
  }
  st->report.rank_deficient[k] = degraded;
}

// ---------------------------------------------------------------------------
// Colour-corrected crops (apply_matrix_rows restricted to the crops, the
// only part of the views the flow and fusion read) + level-0 luma
// (to_luma, frame.cpp:37-50).  grid: (x blocks, 2*n_pairs)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_flow_prepare(const Geometry* __restrict__ g,
                                                      const DevState* __restrict__ st) {
  const int k = blockIdx.y >> 1;
  const int side = blockIdx.y & 1;
  const PairDesc& p = g->pairs[k];
  const int view = side ? p.partner : p.view;
  const double* m = st->mview[view];
  const int n = p.w * p.h;
  const uchar4* raw = p.crop_raw[side];
  uchar4* cor = p.crop_cor[side];
  float* luma = p.pyr[side][0];
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += gridDim.x * blockDim.x) {
    uchar4 c = raw[idx];
    if (c.w) c = apply_matrix(m, c);
    cor[idx] = c;
    if (luma) luma[idx] = c.w ? luma601(c.x, c.y, c.z) : 0.0f;
  }
}

// downsample_half, flow.cpp:16-31.  grid: (x blocks, tasks)
__global__ void __launch_bounds__(256) k_pyr_down(const PyrTask* __restrict__ tasks) {
  const PyrTask t = tasks[blockIdx.y];
  const int n = t.w * t.h;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += gridDim.x * blockDim.x) {
    const int y = idx / t.w;
    const int x = idx - y * t.w;
    const int x0 = 2 * x, y0 = 2 * y;
    const int x1 = min(x0 + 1, t.sw - 1), y1 = min(y0 + 1, t.sh - 1);
    const float* s = t.src;
    t.dst[idx] = 0.25f * (s[y0 * t.sw + x0] + s[y0 * t.sw + x1] + s[y1 * t.sw + x0] +
                          s[y1 * t.sw + x1]);
  }
}

// resize_bilinear of both flow components with value_scale = sx for u AND v
// (flow.cpp:33-55, dense_flow quirk at flow.cpp:163-167).
__global__ void __launch_bounds__(256) k_upsample(const UpTask* __restrict__ tasks) {
  const UpTask t = tasks[blockIdx.y];
  const int n = t.w * t.h;
  const int sw = t.w_in, sh = t.h_in;
  const float scale = static_cast<float>(t.w) / static_cast<float>(sw);
  const float fx = t.w > 1 ? static_cast<float>(sw - 1) / static_cast<float>(t.w - 1) : 0.0f;
  const float fy = t.h > 1 ? static_cast<float>(sh - 1) / static_cast<float>(t.h - 1) : 0.0f;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += gridDim.x * blockDim.x) {
    const int y = idx / t.w;
    const int x = idx - y * t.w;
    const float sy = static_cast<float>(y) * fy;
    const int y0 = min(sh - 1, static_cast<int>(sy));
    const int y1 = min(sh - 1, y0 + 1);
    const float ay = sy - static_cast<float>(y0);
    const float sx = static_cast<float>(x) * fx;
    const int x0 = min(sw - 1, static_cast<int>(sx));
    const int x1 = min(sw - 1, x0 + 1);
    const float ax = sx - static_cast<float>(x0);
    {
      const float* s = t.u_in;
      const float top = (1.0f - ax) * s[y0 * sw + x0] + ax * s[y0 * sw + x1];
      const float bot = (1.0f - ax) * s[y1 * sw + x0] + ax * s[y1 * sw + x1];
      t.u_out[idx] = scale * ((1.0f - ay) * top + ay * bot);
    }
    {
      const float* s = t.v_in;
      const float top = (1.0f - ax) * s[y0 * sw + x0] + ax * s[y0 * sw + x1];
      const float bot = (1.0f - ax) * s[y1 * sw + x0] + ax * s[y1 * sw + x1];
      t.v_out[idx] = scale * ((1.0f - ay) * top + ay * bot);
    }
  }
}

// ---------------------------------------------------------------------------
// One warp iteration of refine_level (flow.cpp:84-134), temporally blocked:
// the CTA loads its output tile plus a halo of `sweeps` pixels, computes the
// warped image bw = sample_clamped(b, x+u, y+v) on it, the linearisation
// (ix, iy, it) one pixel in, and then runs all Jacobi sweeps in shared
// memory on a region that shrinks by one pixel per sweep.  Each sweep reads
// only the previous buffer, so the result is bit-identical to the
// reference's full-plane double-buffered passes.
// grid: (tiles x, tiles y, tasks); dynamic smem: 9 planes of the region.
// ---------------------------------------------------------------------------
constexpr int kHsTX = 32;
constexpr int kHsTY = 16;

__global__ void __launch_bounds__(256) k_hs_iter(const HsTask* __restrict__ tasks, int sweeps,
                                                 float alpha2) {
  const HsTask t = tasks[blockIdx.z];
  const int tx0 = blockIdx.x * kHsTX, ty0 = blockIdx.y * kHsTY;
  if (tx0 >= t.w || ty0 >= t.h) return;
  const int w = t.w, h = t.h;
  const int H = sweeps;
  const int tx1 = min(w, tx0 + kHsTX), ty1 = min(h, ty0 + kHsTY);
  const int rx0 = max(0, tx0 - H), ry0 = max(0, ty0 - H);
  const int rx1 = min(w, tx1 + H), ry1 = min(h, ty1 + H);
  const int RW = rx1 - rx0, RH = ry1 - ry0;
  const int RN = RW * RH;
  extern __shared__ float smem[];
  float* su0 = smem;
  float* sv0 = su0 + RN;
  float* su1 = sv0 + RN;
  float* sv1 = su1 + RN;
  float* sbw = sv1 + RN;
  float* sgx = sbw + RN;
  float* sgy = sgx + RN;
  float* sc = sgy + RN;
  float* sden = sc + RN;
  const int tid = threadIdx.x, nt = blockDim.x;

  // 1) flow at the start of this warp (u0, v0) and the warped image bw
  for (int i = tid; i < RN; i += nt) {
    const int ly = i / RW, lx = i - ly * RW;
    const int x = rx0 + lx, y = ry0 + ly;
    float u = 0.0f, v = 0.0f;
    if (!t.zero_in) {
      u = t.u_in[y * w + x];
      v = t.v_in[y * w + x];
    }
    su0[i] = u;
    sv0[i] = v;
    sbw[i] = sample_clamped(t.b, w, h, static_cast<float>(x) + u, static_cast<float>(y) + v);
  }
  __syncthreads();
  // 2) linearisation over the region shrunk by one (flow.cpp:95-108)
  {
    const int ex = H - 1;
    const int cx0 = max(0, tx0 - ex), cy0 = max(0, ty0 - ex);
    const int cx1 = min(w, tx1 + ex), cy1 = min(h, ty1 + ex);
    const int CW = cx1 - cx0, CN = CW * (cy1 - cy0);
    for (int i = tid; i < CN; i += nt) {
      const int cy = i / CW;
      const int x = cx0 + (i - cy * CW), y = cy0 + cy;
      const int ym = max(0, y - 1), yp = min(h - 1, y + 1);
      const int xm = max(0, x - 1), xp = min(w - 1, x + 1);
      const float* a = t.a;
      const float gx = 0.25f * (__ldg(a + y * w + xp) - __ldg(a + y * w + xm) +
                                sbw[(y - ry0) * RW + (xp - rx0)] - sbw[(y - ry0) * RW + (xm - rx0)]);
      const float gy = 0.25f * (__ldg(a + yp * w + x) - __ldg(a + ym * w + x) +
                                sbw[(yp - ry0) * RW + (x - rx0)] - sbw[(ym - ry0) * RW + (x - rx0)]);
      const float it = sbw[(y - ry0) * RW + (x - rx0)] - __ldg(a + y * w + x);
      const int li = (y - ry0) * RW + (x - rx0);
      sgx[li] = gx;
      sgy[li] = gy;
      // Residual constant of the Jacobi update: c = it - gx*u0 - gy*v0 and
      // denom = alpha2 + gx*gx + gy*gy do not change across sweeps.
      sc[li] = it - gx * su0[li] - gy * sv0[li];
      sden[li] = alpha2 + gx * gx + gy * gy;
    }
  }
  __syncthreads();
  // 3) Jacobi sweeps (flow.cpp:109-134)
  float* ucur = su0;
  float* vcur = sv0;
  float* unxt = su1;
  float* vnxt = sv1;
  for (int s = 1; s <= sweeps; ++s) {
    const int ex = sweeps - s;
    const int cx0 = max(0, tx0 - ex), cy0 = max(0, ty0 - ex);
    const int cx1 = min(w, tx1 + ex), cy1 = min(h, ty1 + ex);
    const int CW = cx1 - cx0, CN = CW * (cy1 - cy0);
    for (int i = tid; i < CN; i += nt) {
      const int cy = i / CW;
      const int x = cx0 + (i - cy * CW), y = cy0 + cy;
      const int lym = (max(0, y - 1) - ry0) * RW, lyp = (min(h - 1, y + 1) - ry0) * RW;
      const int ly = (y - ry0) * RW;
      const int lx = x - rx0, lxm = max(0, x - 1) - rx0, lxp = min(w - 1, x + 1) - rx0;
      const float ubar = 0.25f * (ucur[ly + lxm] + ucur[ly + lxp] + ucur[lym + lx] + ucur[lyp + lx]);
      const float vbar = 0.25f * (vcur[ly + lxm] + vcur[ly + lxp] + vcur[lym + lx] + vcur[lyp + lx]);
      const int li = ly + lx;
      const float gx = sgx[li], gy = sgy[li];
      const float common = (gx * ubar + gy * vbar + sc[li]) / sden[li];
      unxt[li] = ubar - gx * common;
      vnxt[li] = vbar - gy * common;
    }
    __syncthreads();
    float* tu = ucur;
    ucur = unxt;
    unxt = tu;
    float* tv = vcur;
    vcur = vnxt;
    vnxt = tv;
  }
  // 4) write the tile
  const int TW = tx1 - tx0, TN = TW * (ty1 - ty0);
  for (int i = tid; i < TN; i += nt) {
    const int yy = i / TW;
    const int x = tx0 + (i - yy * TW), y = ty0 + yy;
    const int li = (y - ry0) * RW + (x - rx0);
    float u = ucur[li], v = vcur[li];
    if (t.zero_invalid) {
      // dense_flow zeroes the field where either input is invalid
      // (flow.cpp:178-185)
      if (!t.mask_a[y * w + x].w || !t.mask_b[y * w + x].w) {
        u = 0.0f;
        v = 0.0f;
      }
    }
    t.u_out[y * w + x] = u;
    t.v_out[y * w + x] = v;
  }
}

// ---------------------------------------------------------------------------
// Canvas pass: for every canvas pixel, the warped reference view, then the
// compose_panorama fold over pairs (pipeline.cpp:326-333, flow.cpp:324-357)
// with the colour-corrected warped view (apply_matrix_rows, pipeline.cpp:296)
// and, inside each overlap, the flow-displaced fusion of flow_fuse
// (flow.cpp:282-322) evaluated on demand.  Also the balance histogram of
// the composed panorama (compute_histogram, histogram.cpp:5-18).
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool fused_pixel(const Geometry* __restrict__ g, const PairDesc& p,
                                            int dx, int dy, uchar4& out) {
  const int i = dy * p.w + dx;
  const float ti = p.theta_i[i];
  const float tj = 1.0f - ti;  // BlendWeights::theta_j (flow.cpp:276)
  const float wi = g->weighting == 0 ? ti : tj;
  const float wj = g->weighting == 0 ? tj : ti;
  float ri, gi, bi, rj, gj, bj;
  const bool vi = sample_crop(p.crop_cor[0], p.w, p.h,
                              static_cast<double>(static_cast<float>(dx) + wi * p.flow_u[0][i]),
                              static_cast<double>(static_cast<float>(dy) + wi * p.flow_v[0][i]),
                              ri, gi, bi);
  const bool vj = sample_crop(p.crop_cor[1], p.w, p.h,
                              static_cast<double>(static_cast<float>(dx) + wj * p.flow_u[1][i]),
                              static_cast<double>(static_cast<float>(dy) + wj * p.flow_v[1][i]),
                              rj, gj, bj);
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
  out = make_uchar4(quantize_d(r), quantize_d(gg), quantize_d(b), 1);
  return true;
}

__global__ void __launch_bounds__(256) k_canvas(const Geometry* __restrict__ g,
                                                DevState* __restrict__ st,
                                                uchar4* __restrict__ pano, long long n_px) {
  __shared__ unsigned int hist[3][256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    hist[0][i] = 0;
    hist[1][i] = 0;
    hist[2][i] = 0;
  }
  __syncthreads();
  const int cw = g->canvas_w;
  const int ref = g->reference;
  const ViewDesc& vr = g->views[ref];
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < n_px;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int y = static_cast<int>(idx / cw);
    const int x = static_cast<int>(idx - static_cast<long long>(y) * cw);
    const double X = static_cast<double>(x) + g->offx;
    const double Y = static_cast<double>(y) + g->offy;
    uchar4 pv = make_uchar4(0, 0, 0, 0);
    if (x >= vr.bbox[0] && x < vr.bbox[2] && y >= vr.bbox[1] && y < vr.bbox[3])
      pv = warp_sample(vr, g->frames[ref], X, Y);
    for (int k = 0; k < g->n_pairs; ++k) {
      const PairDesc& p = g->pairs[k];
      const ViewDesc& vv = g->views[p.view];
      if (x < vv.bbox[0] || x >= vv.bbox[2] || y < vv.bbox[1] || y >= vv.bbox[3]) continue;
      uchar4 q = warp_sample(vv, g->frames[p.view], X, Y);
      if (!q.w) continue;
      if (pv.w) {
        const int dx = x - p.x0, dy = y - p.y0;
        if (dx >= 0 && dy >= 0 && dx < p.w && dy < p.h) {
          uchar4 f;
          if (fused_pixel(g, p, dx, dy, f)) pv = f;
        }
      } else {
        pv = apply_matrix(st->mview[p.view], q);
      }
    }
    pano[idx] = pv;
    if (pv.w) {
      atomicAdd(&hist[0][pv.x], 1u);
      atomicAdd(&hist[1][pv.y], 1u);
      atomicAdd(&hist[2][pv.z], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    for (int c = 0; c < 3; ++c)
      if (hist[c][i]) atomicAdd(&st->pano_hist[c][i], hist[c][i]);
}

// ---------------------------------------------------------------------------
// Global balancing on one CTA: find_thresholds (color_balance.cpp:8-38),
// history push (pipeline.cpp:340-345), smooth_thresholds
// (color_balance.cpp:40-63), build_curve (color_balance.cpp:65-104).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_balance(const Geometry* __restrict__ g,
                                                 DevState* __restrict__ st) {
  __shared__ unsigned int hist[3][256];
  __shared__ int sm1[3], sm2[3];
  __shared__ int ok;
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    for (int c = 0; c < 3; ++c) {
      hist[c][i] = st->pano_hist[c][i];
      st->pano_hist[c][i] = 0;
    }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long total = 0;
    for (int v = 0; v < 256; ++v) total += hist[0][v];
    ok = 0;
    st->report.frame_index = st->frame_counter;
    if (total != 0) {
      int m1[3], m2[3];
      const double tot = static_cast<double>(total);
      for (int c = 0; c < 3; ++c) {
        unsigned long long run = 0;
        int a = 255, b = 255;
        bool h1 = false;
        for (int v = 0; v < 256; ++v) {
          run += hist[c][v];
          const double cdf = static_cast<double>(run) / tot;
          if (!h1 && cdf >= g->lambda) {
            a = v;
            h1 = true;
          }
          if (cdf >= 1.0 - g->lambda) {
            b = v;
            break;
          }
        }
        m1[c] = a;
        m2[c] = b;
      }
      BalanceState& bs = st->balance;
      if (bs.n == 3) {
        for (int i = 0; i < 2; ++i)
          for (int c = 0; c < 3; ++c) {
            bs.m1[i][c] = bs.m1[i + 1][c];
            bs.m2[i][c] = bs.m2[i + 1][c];
          }
        bs.n = 2;
      }
      for (int c = 0; c < 3; ++c) {
        bs.m1[bs.n][c] = m1[c];
        bs.m2[bs.n][c] = m2[c];
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
    st->frame_counter++;
  }
  __syncthreads();
  // build_curve: one thread per level, all three channels
  for (int v = threadIdx.x; v < 256; v += blockDim.x) {
    for (int c = 0; c < 3; ++c) {
      unsigned char out = static_cast<unsigned char>(v);
      if (ok) {
        const int m1 = sm1[c], m2 = sm2[c];
        const double tb = g->target_black, tw = g->target_white;
        const double x = static_cast<double>(v);
        double val;
        if (m1 >= m2) {
          val = tb + (tw - tb) * (x / 255.0);
        } else {
          const double lm1 = tb + (tw - tb) * (static_cast<double>(m1) / 255.0);
          const double lm2 = tb + (tw - tb) * (static_cast<double>(m2) / 255.0);
          if (x <= m1) {
            val = (m1 == 0) ? tb : tb + (lm1 - tb) * pow(x / m1, g->gamma_dark);
          } else if (x >= m2) {
            val = (m2 == 255) ? tw : lm2 + (tw - lm2) * pow((x - m2) / (255.0 - m2), g->gamma_bright);
          } else {
            val = lm1 + (lm2 - lm1) * (x - m1) / (m2 - m1);
          }
        }
        out = quantize_d(val);
      }
      st->lut[c][v] = out;
    }
  }
}

// apply_tone_rows (pipeline.cpp:84-96) + conversion to the reference's Frame
// layout (RGB8 interleaved + 0/1 mask).  4 pixels per thread: one 16-byte
// uchar4x4 load, three 4-byte RGB stores, one 4-byte mask store.
__global__ void __launch_bounds__(256) k_tone(const DevState* __restrict__ st,
                                              const uchar4* __restrict__ pano, long long n_px,
                                              std::uint8_t* __restrict__ out_rgb,
                                              std::uint8_t* __restrict__ out_mask) {
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
__global__ void __launch_bounds__(256) k_warp_view(const Geometry* __restrict__ g, int view,
                                                   const std::uint8_t* __restrict__ frame,
                                                   std::uint8_t* __restrict__ rgb,
                                                   std::uint8_t* __restrict__ mask) {
  const ViewDesc& v = g->views[view];
  const long long n = static_cast<long long>(g->canvas_w) * g->canvas_h;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < n;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int y = static_cast<int>(idx / g->canvas_w);
    const int x = static_cast<int>(idx - static_cast<long long>(y) * g->canvas_w);
    const uchar4 o = warp_sample(v, frame, static_cast<double>(x) + g->offx,
                                 static_cast<double>(y) + g->offy);
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
__global__ void __launch_bounds__(256) k_warp_mask(const Geometry* __restrict__ g, int view,
                                                   std::uint8_t* __restrict__ mask) {
  const ViewDesc& v = g->views[view];
  const long long n = static_cast<long long>(g->canvas_w) * g->canvas_h;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < n;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int y = static_cast<int>(idx / g->canvas_w);
    const int x = static_cast<int>(idx - static_cast<long long>(y) * g->canvas_w);
    const double X = static_cast<double>(x) + g->offx;
    const double Y = static_cast<double>(y) + g->offy;
    const double* m = v.inv;
    const double sx0 = (m[0] * X + m[1] * Y) + m[2];
    const double sy0 = (m[3] * X + m[4] * Y) + m[5];
    const double sz0 = (m[6] * X + m[7] * Y) + m[8];
    unsigned char ok = 0;
    if (!(fabs(sz0) < 1e-12)) {
      const double sx = sx0 / sz0, sy = sy0 / sz0;
      const double fx0 = floor(sx), fy0 = floor(sy);
      const int x0 = static_cast<int>(fx0), y0 = static_cast<int>(fy0);
      const double ax = sx - fx0, ay = sy - fy0;
      for (int j = 0; j < 2 && !ok; ++j)
        for (int i = 0; i < 2 && !ok; ++i) {
          const double w = (i ? ax : 1.0 - ax) * (j ? ay : 1.0 - ay);
          const unsigned xx = static_cast<unsigned>(x0) + i, yy = static_cast<unsigned>(y0) + j;
          if (w > 0.0 && xx < static_cast<unsigned>(v.width) && yy < static_cast<unsigned>(v.height))
            ok = 1;
        }
    }
    mask[idx] = ok;
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

void launch_crop_warp(const Geometry* g, int n_pairs, int max_crop_px, cudaStream_t s) {
  dim3 grid(blocks_for(max_crop_px), 2 * n_pairs);
  k_crop_warp<<<grid, 256, 0, s>>>(g);
}

void launch_pair_stats(const Geometry* g, DevState* st, const int* list, int n, int max_crop_px,
                       cudaStream_t s) {
  dim3 grid(blocks_for(max_crop_px, 256 * 16, 512), n);
  k_pair_stats<<<grid, 256, 0, s>>>(g, st, list);
}

void launch_pair_solve(const Geometry* g, DevState* st, const int* list, int n, cudaStream_t s) {
  k_pair_solve<<<n, 256, 0, s>>>(g, st, list);
}

void launch_flow_prepare(const Geometry* g, DevState* st, int n_pairs, int max_crop_px,
                         cudaStream_t s) {
  dim3 grid(blocks_for(max_crop_px), 2 * n_pairs);
  k_flow_prepare<<<grid, 256, 0, s>>>(g, st);
}

void launch_pyr_down(const PyrTask* tasks, int n, int max_px, cudaStream_t s) {
  dim3 grid(blocks_for(max_px), n);
  k_pyr_down<<<grid, 256, 0, s>>>(tasks);
}

void launch_upsample(const UpTask* tasks, int n, int max_px, cudaStream_t s) {
  dim3 grid(blocks_for(max_px), n);
  k_upsample<<<grid, 256, 0, s>>>(tasks);
}

size_t hs_smem_bytes(int sweeps) {
  return static_cast<size_t>(9) * (kHsTX + 2 * sweeps) * (kHsTY + 2 * sweeps) * sizeof(float);
}

cudaError_t prepare_hs(int sweeps) {
  return cudaFuncSetAttribute(k_hs_iter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(hs_smem_bytes(sweeps)));
}

void launch_hs_iter(const HsTask* tasks, int n, int max_w, int max_h, int sweeps, float alpha2,
                    cudaStream_t s) {
  const size_t smem = hs_smem_bytes(sweeps);
  dim3 grid((max_w + kHsTX - 1) / kHsTX, (max_h + kHsTY - 1) / kHsTY, n);
  k_hs_iter<<<grid, 256, smem, s>>>(tasks, sweeps, alpha2);
}

void launch_canvas(const Geometry* g, DevState* st, uchar4* pano, long long n_px, int num_sms,
                   cudaStream_t s) {
  const int blocks = static_cast<int>(
      std::min<long long>(static_cast<long long>(num_sms) * 8, (n_px + 255) / 256));
  k_canvas<<<blocks < 1 ? 1 : blocks, 256, 0, s>>>(g, st, pano, n_px);
}

void launch_balance(const Geometry* g, DevState* st, cudaStream_t s) {
  k_balance<<<1, 256, 0, s>>>(g, st);
}

void launch_tone(const DevState* st, const uchar4* pano, long long n_px, std::uint8_t* out_rgb,
                 std::uint8_t* out_mask, cudaStream_t s) {
  k_tone<<<blocks_for(n_px / 4 + 1, 256, 148 * 16), 256, 0, s>>>(st, pano, n_px, out_rgb,
                                                                  out_mask);
}

void launch_warp_view(const Geometry* g, int view, const std::uint8_t* frame, std::uint8_t* rgb,
                      std::uint8_t* mask, cudaStream_t s) {
  k_warp_view<<<148 * 8, 256, 0, s>>>(g, view, frame, rgb, mask);
}

void launch_warp_mask(const Geometry* g, int view, std::uint8_t* mask, cudaStream_t s) {
  k_warp_mask<<<148 * 8, 256, 0, s>>>(g, view, mask);
}

}  // namespace stitch_b200_dev
