// color_kernels.cu -- 3D-M spatio-temporal colour transfer (transfer_step,
// /root/reference/proj/src/color_transfer.cpp:133-191, as driven by
// process_frame, pipeline.cpp:279-300), a statistics launch and a solve
// launch per pair depth.
//
// Single HBM pass over the jointly valid overlap pixels reduced to integer
// tables (source/reference histograms and the conditional sums
// S_{a|b}[v] = sum_{x_b = v} x_a), from which the specification LUT and the
// exact moments X^T X and X^T Y of the LUT-revised rows follow:
//   X^T X[a][a] = sum_v v^2 h_a[v],        X^T X[a][b] = sum_v v S_{a|b}[v]
//   X^T Y[a][a] = sum_v v LUT_a[v] h_a[v], X^T Y[a][b] = sum_v LUT_b[v] S_{a|b}[v]
// All entries are integers < 2^53, so the window sum (ring of <= 3 frames)
// is bit-identical to the reference's stacked-row normal equations.
// k_pair_solve then solves each pair (or, STITCH_B200_COLOR_SPLIT=0, the
// last CTA of each pair's statistics, elected by a grid-wide counter).
#include <cuda_runtime.h>

#include <algorithm>

#include "device_math.cuh"
#include "kernels.cuh"

namespace stitch_b200_dev {

__device__ __forceinline__ int sidx(int a, int b) { return a * 2 + (b > a ? b - 1 : b); }

// The per-pair solve, one 256-thread CTA per pair (k_pair_solve, or the
// pair's last statistics CTA):
// histogram_specification (color_transfer.cpp:28-55), revised-row moments,
// TransferWindow push (color_transfer.cpp:16-21), solve_color_matrix with
// the rank guard (color_transfer.cpp:73-99), and the degrade rules of
// process_frame (pipeline.cpp:282-293).
__device__ void pair_solve(const PairDesc& p, int k, DevState* __restrict__ st) {
  __shared__ unsigned char lut[3][256];
  __shared__ unsigned long long cref[3][256];
  PairStats& in = st->stats[k];
  const int v = threadIdx.x;  // level owned by this thread
  const unsigned long long n = in.n;
  unsigned int hs[3], hr[3];
  unsigned long long ss[6];
  for (int c = 0; c < 3; ++c) {
    hs[c] = in.hs[c][v];
    hr[c] = in.hr[c][v];
    in.hs[c][v] = 0;  // reset the accumulators for the next frame
    in.hr[c][v] = 0;
  }
  for (int c = 0; c < 6; ++c) {
    ss[c] = in.s[c][v];
    in.s[c][v] = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) in.n = 0;
  if (n == 0) {
    // EmptyRegion from transfer_step: identity M, window untouched
    if (threadIdx.x == 0) {
      for (int i = 0; i < 9; ++i) {
        const double e = (i % 4 == 0) ? 1.0 : 0.0;
        st->mview[p.view][i] = e;
        st->report.m[k][i] = e;
      }
      st->report.rank_deficient[k] = 1;
    }
    return;
  }
  // LUT[c][v] = smallest u in [0, 255) with cum_ref[u] >= cum_src[v], else
  // 255 -- the reference's monotone scan (both histograms count the same n
  // jointly valid pixels, so its cross-multiplied compare reduces to this).
  // The six inclusive prefix sums (3 reference, 3 source) are scanned
  // together: warp shuffles, one exchange of the warp totals.
  __shared__ unsigned long long wsum6[8][6];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long sc[6];
  for (int c = 0; c < 3; ++c) {
    sc[c] = hr[c];
    sc[3 + c] = hs[c];
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1)
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, sc[j], o);
      if (lane >= o) sc[j] += y;
    }
  if (lane == 31)
    for (int j = 0; j < 6; ++j) wsum6[wid][j] = sc[j];
  __syncthreads();
  for (int i = 0; i < wid; ++i)
    for (int j = 0; j < 6; ++j) sc[j] += wsum6[i][j];
  unsigned long long csrc[3];
  for (int c = 0; c < 3; ++c) {
    cref[c][v] = sc[c];
    csrc[c] = sc[3 + c];
  }
  __syncthreads();
  for (int c = 0; c < 3; ++c) {
    int lo = 0, hi = 255;  // search in [0, 255)
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (cref[c][mid] < csrc[c])
        lo = mid + 1;
      else
        hi = mid;
    }
    lut[c][v] = static_cast<unsigned char>(lo);
  }
  __syncthreads();
  // exact integer moments: every thread's 18 terms, reduced per warp by
  // shuffles, the 8 warp partials summed below (integer: any order)
  __shared__ unsigned long long wmom[8][18];
  const unsigned long long vv = static_cast<unsigned long long>(v);
#pragma unroll
  for (int q = 0; q < 18; ++q) {
    const int which = q / 9, a = (q % 9) / 3, b = q % 3;
    unsigned long long x;
    if (which == 0)
      x = (a == b) ? vv * vv * hs[a] : vv * ss[sidx(a, b)];
    else
      x = (a == b) ? vv * lut[a][v] * hs[a] : static_cast<unsigned long long>(lut[b][v]) * ss[sidx(a, b)];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) wmom[wid][q] = x;
  }
  __syncthreads();
  // TransferWindow push (newest first, capacity-clamped) and the window
  // sums, one thread per moment entry (18) plus one for the counts: the
  // entries are independent, so the global reads and writes of the ring
  // overlap instead of running as one thread's dependent chain
  PairWindow& w = st->windows[k];
  const int size = w.size < w.capacity ? w.size + 1 : w.capacity;
  __shared__ unsigned long long wsum[19];
  if (threadIdx.x < 19) {
    const int q = threadIdx.x;
    unsigned long long cur;
    if (q < 18) {
      cur = 0;
      for (int i = 0; i < 8; ++i) cur += wmom[i][q];
    } else {
      cur = n;
    }
    auto slot = [&](int e) -> unsigned long long& {
      return q < 9 ? w.e[e].xtx[q] : (q < 18 ? w.e[e].xty[q - 9] : w.e[e].n);
    };
    unsigned long long old[3];
    for (int e = 0; e + 1 < size; ++e) old[e] = slot(e);
    unsigned long long sum = cur;
    for (int e = size - 1; e > 0; --e) {
      slot(e) = old[e - 1];
      sum += old[e - 1];
    }
    slot(0) = cur;
    wsum[q] = sum;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  w.size = size;
  unsigned long long sx[9], sy[9];
  for (int i = 0; i < 9; ++i) {
    sx[i] = wsum[i];
    sy[i] = wsum[9 + i];
  }
  const unsigned long long total = wsum[18];
  double normal[9], xty[9], m[9], sv[3];
  for (int i = 0; i < 9; ++i) {
    normal[i] = static_cast<double>(sx[i]);
    xty[i] = static_cast<double>(sy[i]);
  }
  // Rank guard (color_transfer.cpp:88-91): sigma_min < 1e-8 sigma_max, with
  // sigma = the eigenvalues of the PSD normal matrix.  The decision is
  // settled without the eigensolve whenever det / tr^3 bounds it with
  // margin: lambda_min / lambda_max >= det / tr^3 (lambda_max <= tr) and
  // <= sqrt(27 det / tr^3) (lambda_max >= tr / 3, lambda_min^2 <= det /
  // lambda_max); det carries a generous rounding bound.  The 2 % margins
  // dwarf the eigensolver's ~1e-15 relative error, so the outcome equals
  // the full cyclic-Jacobi test, which runs only in the narrow band between.
  int rank_ok = -1;
  {
    const double* a = normal;
    const double c0 = a[4] * a[8] - a[5] * a[7];
    const double c1 = a[3] * a[8] - a[5] * a[6];
    const double c2 = a[3] * a[7] - a[4] * a[6];
    const double det = (a[0] * c0 - a[1] * c1) + a[2] * c2;
    const double mag = fabs(a[0]) * (fabs(a[4] * a[8]) + fabs(a[5] * a[7])) +
                       fabs(a[1]) * (fabs(a[3] * a[8]) + fabs(a[5] * a[6])) +
                       fabs(a[2]) * (fabs(a[3] * a[7]) + fabs(a[4] * a[6]));
    const double err = 1e-13 * mag;
    const double tr = (a[0] + a[4]) + a[8];
    const double tr3 = tr * tr * tr;
    if (tr > 0.0 && det - err > 1.02e-8 * tr3) rank_ok = 1;
    else if (tr > 0.0 && 27.0 * (det + err) < 0.98e-16 * tr3) rank_ok = 0;
  }
  if (rank_ok < 0) {
    sym3_eigen(normal, sv);
    rank_ok = sv[2] < 1e-8 * sv[0] ? 0 : 1;
  }
  int degraded = 0;
  if (total < 3 || !rank_ok) {
    for (int i = 0; i < 9; ++i) m[i] = (i % 4 == 0) ? 1.0 : 0.0;  // RankDeficient
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

// Pixels per thread (grid = ceil(n / (256 * kColorPpt)) CTAs per pair): each
// CTA then sees at most 256 * kColorPpt = 2048 pixels, which bounds its
// per-level partial sums (<= 2048 * 255 < 2^19) and counts (<= 2048 < 2^12)
// so a count and a conditional sum share one 32-bit shared counter.
constexpr int kColorPpt = 8;
constexpr int kSumBits = 19;
constexpr unsigned kSumMask = (1u << kSumBits) - 1u;

// grid: (blocks per pair, pairs of this depth); 256 threads.
// Per jointly valid pixel and channel b (bin v = x_b): the count, the sum
// of the lower other channel x_a1 and of the higher one x_a2 land in the
// same bin, so the count and x_a1 share one packed counter
// (count << 19 | sum) and x_a2 gets its own: 6 shared atomics for the
// source side instead of 9, plus 3 for the reference histogram.
// VEC: each thread reads its 8 consecutive pixels of both crops with two
// 16-byte loads per crop, all issued before any use.  ELECT: the pair's
// last CTA performs the solve (else k_pair_solve, launched after).
__device__ __forceinline__ void color_accum(uchar4 a, uchar4 b, bool correct_partner,
                                            const double* mp, unsigned (&pk)[3][256],
                                            unsigned (&s2)[3][256], unsigned (&hr)[3][256],
                                            unsigned& local) {
  if (!a.w || !b.w) return;
  if (correct_partner) b = apply_matrix(mp, b);
  // bin channel 0: a1 = 1, a2 = 2; channel 1: a1 = 0, a2 = 2; channel 2: a1 = 0, a2 = 1
  atomicAdd(&pk[0][a.x], (1u << kSumBits) + a.y);
  atomicAdd(&s2[0][a.x], static_cast<unsigned>(a.z));
  atomicAdd(&pk[1][a.y], (1u << kSumBits) + a.x);
  atomicAdd(&s2[1][a.y], static_cast<unsigned>(a.z));
  atomicAdd(&pk[2][a.z], (1u << kSumBits) + a.x);
  atomicAdd(&s2[2][a.z], static_cast<unsigned>(a.y));
  atomicAdd(&hr[0][b.x], 1u);
  atomicAdd(&hr[1][b.y], 1u);
  atomicAdd(&hr[2][b.z], 1u);
  ++local;
}

__device__ __forceinline__ uchar4 u32_px(unsigned w) {
  return make_uchar4(w & 0xffu, (w >> 8) & 0xffu, (w >> 16) & 0xffu, w >> 24);
}

template <bool ELECT, bool VEC>
__global__ void __launch_bounds__(256) k_pair_color(const Geometry* __restrict__ g,
                                                    DevState* __restrict__ st,
                                                    const int* __restrict__ list) {
  pdl_wait();
  __shared__ unsigned int pk[3][256];  // count << 19 | sum of x_a1, bin x_b
  __shared__ unsigned int s2[3][256];  // sum of x_a2, bin x_b
  __shared__ unsigned int hr[3][256];
  __shared__ unsigned int cnt;
  const int k = list[blockIdx.y];
  const PairDesc& p = g->pairs[k];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    for (int c = 0; c < 3; ++c) {
      pk[c][i] = 0;
      s2[c][i] = 0;
      hr[c][i] = 0;
    }
  }
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  // the partner is already corrected when it is not the reference (chain)
  const bool correct_partner = p.partner != g->reference;
  const double* mp = st->mview[p.partner];
  const int n = p.w * p.h;
  unsigned int local = 0;
  if (VEC) {
    const long long i0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
    if (i0 + 8 <= n) {
      const uint4* qa = reinterpret_cast<const uint4*>(p.crop_raw[0] + i0);
      const uint4* qb = reinterpret_cast<const uint4*>(p.crop_raw[1] + i0);
      const uint4 a0 = __ldg(qa), a1 = __ldg(qa + 1), b0 = __ldg(qb), b1 = __ldg(qb + 1);
      const unsigned wa[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const unsigned wb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int j = 0; j < 8; ++j)
        color_accum(u32_px(wa[j]), u32_px(wb[j]), correct_partner, mp, pk, s2, hr, local);
    } else {
      for (long long i = i0; i < n && i < i0 + 8; ++i)
        color_accum(__ldg(p.crop_raw[0] + i), __ldg(p.crop_raw[1] + i), correct_partner, mp, pk,
                    s2, hr, local);
    }
  } else {
    // 4 pixels per step, their 8 crop loads issued before any use
    constexpr int kB = 4;
    const int stride = gridDim.x * blockDim.x;
    for (int base = blockIdx.x * blockDim.x + threadIdx.x; base < n; base += kB * stride) {
      uchar4 pa[kB], pb[kB];
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        const int idx = base + j * stride;
        pa[j] = make_uchar4(0, 0, 0, 0);
        pb[j] = make_uchar4(0, 0, 0, 0);
        if (idx < n) {
          pa[j] = __ldg(p.crop_raw[0] + idx);
          pb[j] = __ldg(p.crop_raw[1] + idx);
        }
      }
#pragma unroll
      for (int j = 0; j < kB; ++j) color_accum(pa[j], pb[j], correct_partner, mp, pk, s2, hr, local);
    }
  }
  atomicAdd(&cnt, local);
  __syncthreads();
  if (!ELECT) pdl_trigger();  // only the flush of the tables remains
  PairStats& out = st->stats[k];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    for (int c = 0; c < 3; ++c) {
      const unsigned w = pk[c][i];
      const unsigned count = w >> kSumBits, sum1 = w & kSumMask, sum2 = s2[c][i];
      const int a1 = c == 0 ? 1 : 0, a2 = c == 2 ? 1 : 2;
      if (count) atomicAdd(&out.hs[c][i], count);
      if (hr[c][i]) atomicAdd(&out.hr[c][i], hr[c][i]);
      if (sum1) atomicAdd(&out.s[sidx(a1, c)][i], static_cast<unsigned long long>(sum1));
      if (sum2) atomicAdd(&out.s[sidx(a2, c)][i], static_cast<unsigned long long>(sum2));
    }
  }
  if (threadIdx.x == 0 && cnt) atomicAdd(&out.n, static_cast<unsigned long long>(cnt));
  if (!ELECT) return;
  // last CTA of this pair performs the solve
  if (!elect_last_cta(&st->pair_done[k], gridDim.x)) return;
  if (threadIdx.x == 0) st->pair_done[k] = 0;
  pair_solve(p, k, st);
}

// the solves of one pair depth after its statistics launch (ELECT = false)
__global__ void __launch_bounds__(256) k_pair_solve(const Geometry* __restrict__ g,
                                                    DevState* __restrict__ st,
                                                    const int* __restrict__ list) {
  pdl_wait();
  const int k = list[blockIdx.x];
  pair_solve(g->pairs[k], k, st);
}

static inline int blocks_for(long long n, int per, int cap) {
  long long b = (n + per - 1) / per;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return static_cast<int>(b);
}

int launch_pair_color(const Geometry* g, DevState* st, const int* list, int n, int max_crop_px,
                      cudaStream_t s) {
  // no cap on the CTA count: the packed counters need <= 256 * kColorPpt
  // pixels per CTA (measured: 16 or 32 pixels per thread are not faster)
  dim3 grid(blocks_for(max_crop_px, 256 * kColorPpt, 1 << 30), n);
  // Each thread reads its 8 consecutive pixels with 16-byte loads, and the
  // solve runs as its own launch after the statistics: the statistics CTAs
  // exit right after their flush instead of waiting for it behind a fence
  // (the last-CTA election), which frees the SMs for the other frames in
  // flight.  Measured at C2: 897.0 -> 903.9 frames/s, statistics + solve
  // 0.058 -> 0.054 ms per frame (scripts/exp22.sh).  STITCH_B200_COLOR_VEC=0
  // / STITCH_B200_COLOR_SPLIT=0 select the strided loads / the last-CTA solve.
  static const int vec = env_int("STITCH_B200_COLOR_VEC", 1);
  static const int split = env_int("STITCH_B200_COLOR_SPLIT", 1);
  if (split) {
    if (vec)
      k_pair_color<false, true><<<grid, 256, 0, s>>>(g, st, list);
    else
      k_pair_color<false, false><<<grid, 256, 0, s>>>(g, st, list);
    k_pair_solve<<<n, 256, 0, s>>>(g, st, list);
    return 2;
  }
  if (vec)
    k_pair_color<true, true><<<grid, 256, 0, s>>>(g, st, list);
  else
    k_pair_color<true, false><<<grid, 256, 0, s>>>(g, st, list);
  return 1;
}

}  // namespace stitch_b200_dev
