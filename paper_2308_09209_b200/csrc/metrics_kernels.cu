// metrics_kernels.cu -- the paper's quality metrics on the device (PSNR and
// SSIM of the colour transfer, Tables 2-3; /root/reference/proj/src/
// metrics.cpp:9-155): on a context's overlap crops of the last frame
// (stitch_b200_pair_quality) or on two frames (stitch_b200_psnr / _ssim).
//
// Parity: PSNR's squared-error sum is an integer (exact in any order; the
// reference's double running sum of d*d is exact below 2^53), the final
// 10*log10 runs on the host with the reference's libm; SSIM evaluates every
// filter tap and window term in the reference's order in FP64 (no FMA), and
// the mean is a single ordered running sum over window positions, so both
// equal the reference's values bit for bit.
#include <cuda_runtime.h>

#include <map>
#include <mutex>

#include <cmath>
#include <cstdint>
#include <vector>

#include "kernels.cuh"

namespace stitch_b200_dev {

constexpr int kSsimWin = 11, kSsimR = 5;

struct SsimKernel {
  double k[kSsimWin];
};

// gaussian_kernel (metrics.cpp:40-49), host libm like the reference
static SsimKernel ssim_kernel() {
  SsimKernel g;
  double sum = 0.0;
  for (int i = 0; i < kSsimWin; ++i) {
    const double d = i - (kSsimWin - 1) / 2.0;
    g.k[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
    sum += g.k[i];
  }
  for (double& v : g.k) v /= sum;
  return g;
}

// RGB8 (+ optional 0/1 mask) -> uchar4 (r, g, b, valid)
__global__ void __launch_bounds__(256) k_pack_rgba(const std::uint8_t* __restrict__ rgb,
                                                   const std::uint8_t* __restrict__ mask, int n,
                                                   uchar4* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = make_uchar4(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2], mask ? (mask[i] ? 1 : 0) : 1);
}

// psnr (metrics.cpp:9-31): integer squared-error sum and count over the
// jointly valid pixels.  acc[0] = sse, acc[1] = n.
__global__ void __launch_bounds__(256) k_psnr_sse(const uchar4* __restrict__ a,
                                                  const uchar4* __restrict__ b, int n,
                                                  unsigned long long* __restrict__ acc) {
  unsigned long long sse = 0, cnt = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uchar4 p = a[i], q = b[i];
    if (!p.w || !q.w) continue;
    const int d0 = static_cast<int>(p.x) - q.x, d1 = static_cast<int>(p.y) - q.y,
              d2 = static_cast<int>(p.z) - q.z;
    sse += static_cast<unsigned long long>(d0 * d0 + d1 * d1 + d2 * d2);
    ++cnt;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sse += __shfl_xor_sync(0xffffffffu, sse, o);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  if ((threadIdx.x & 31) == 0 && cnt) {
    atomicAdd(acc, sse);
    atomicAdd(acc + 1, cnt);
  }
}

// ssim (metrics.cpp:83-155), horizontal pass of gauss_filter on the five
// planes la, lb, la^2, lb^2, la*lb (luma of jointly valid pixels, else 0),
// plus the horizontal 11-tap count of jointly valid pixels.
__global__ void __launch_bounds__(256) k_ssim_h(const uchar4* __restrict__ a,
                                                const uchar4* __restrict__ b, int w, int h,
                                                const SsimKernel g, double* __restrict__ tmp,
                                                int* __restrict__ hcnt) {
  const long long n = static_cast<long long>(w) * h;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int y = static_cast<int>(i / w), x = static_cast<int>(i - static_cast<long long>(y) * w);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0;
    int c = 0;
    if (x >= kSsimR && x < w - kSsimR) {
      for (int t = 0; t < kSsimWin; ++t) {
        const long long j = i - kSsimR + t;
        const uchar4 p = a[j], q = b[j];
        const bool v = p.w && q.w;
        const double la = v ? 0.299 * p.x + 0.587 * p.y + 0.114 * p.z : 0.0;
        const double lb = v ? 0.299 * q.x + 0.587 * q.y + 0.114 * q.z : 0.0;
        s0 += g.k[t] * la;
        s1 += g.k[t] * lb;
        s2 += g.k[t] * (la * la);
        s3 += g.k[t] * (lb * lb);
        s4 += g.k[t] * (la * lb);
        c += v;
      }
    }
    tmp[i] = s0;
    tmp[n + i] = s1;
    tmp[2 * n + i] = s2;
    tmp[3 * n + i] = s3;
    tmp[4 * n + i] = s4;
    hcnt[i] = c;
  }
}

// vertical pass + the per-window SSIM term for interior positions whose
// support is fully jointly valid; term[i] / valid[i] in row-major order.
__global__ void __launch_bounds__(256) k_ssim_v(const double* __restrict__ tmp,
                                                const int* __restrict__ hcnt, int w, int h,
                                                const SsimKernel g, double* __restrict__ term,
                                                std::uint8_t* __restrict__ valid) {
  const long long n = static_cast<long long>(w) * h;
  const double c1 = (0.01 * 255.0) * (0.01 * 255.0);
  const double c2 = (0.03 * 255.0) * (0.03 * 255.0);
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int y = static_cast<int>(i / w), x = static_cast<int>(i - static_cast<long long>(y) * w);
    bool ok = x >= kSsimR && x < w - kSsimR && y >= kSsimR && y < h - kSsimR;
    double t = 0.0;
    if (ok) {
      int cnt = 0;
      double m0 = 0.0, m1 = 0.0, m2 = 0.0, m3 = 0.0, m4 = 0.0;
      for (int k = 0; k < kSsimWin; ++k) {
        const long long j = i + static_cast<long long>(k - kSsimR) * w;
        m0 += g.k[k] * tmp[j];
        m1 += g.k[k] * tmp[n + j];
        m2 += g.k[k] * tmp[2 * n + j];
        m3 += g.k[k] * tmp[3 * n + j];
        m4 += g.k[k] * tmp[4 * n + j];
        cnt += hcnt[j];
      }
      ok = cnt == kSsimWin * kSsimWin;
      if (ok) {
        const double ma = m0, mb = m1;
        const double va = m2 - ma * ma;
        const double vb = m3 - mb * mb;
        const double cov = m4 - ma * mb;
        const double num = (2.0 * ma * mb + c1) * (2.0 * cov + c2);
        const double den = (ma * ma + mb * mb + c1) * (va + vb + c2);
        t = num / den;
      }
    }
    term[i] = t;
    valid[i] = ok ? 1 : 0;
  }
}

// The reference's running sum over window positions, in row-major order
// (metrics.cpp:140-150): one lane adds the terms of the fully valid windows
// in order (FP64, so the rounding sequence is the reference's).
// Same running sum, with the loads off the sum's critical path: warps 1..15
// stage chunk c + 1 of the terms (and their window-validity flags) in shared
// memory while lane 0 of warp 0 adds chunk c in order, so the sum is bound by
// the dependent DADD chain instead of one global round trip per 32 terms.
constexpr int kSumChunk = 2048;

__global__ void __launch_bounds__(512) k_ssim_sum_staged(const double* __restrict__ term,
                                                         const std::uint8_t* __restrict__ valid,
                                                         long long n, double* __restrict__ out_sum,
                                                         long long* __restrict__ out_cnt) {
  __shared__ double st[2][kSumChunk];
  __shared__ std::uint8_t sv[2][kSumChunk];
  const int warp = threadIdx.x >> 5;
  const long long nchunks = (n + kSumChunk - 1) / kSumChunk;
  auto stage = [&](long long c, int buf) {
    const long long base = c * kSumChunk;
    for (int i = threadIdx.x - 32; i < kSumChunk; i += blockDim.x - 32) {
      const long long k = base + i;
      const bool ok = k < n && valid[k];
      sv[buf][i] = ok ? 1 : 0;
      st[buf][i] = ok ? term[k] : 0.0;
    }
  };
  if (warp != 0 && nchunks > 0) stage(0, 0);
  __syncthreads();
  double sum = 0.0;
  long long cnt = 0;
  for (long long c = 0; c < nchunks; ++c) {
    const int buf = static_cast<int>(c & 1);
    if (warp != 0) {
      if (c + 1 < nchunks) stage(c + 1, buf ^ 1);
    } else if (threadIdx.x == 0) {
      const int m = static_cast<int>(n - c * kSumChunk < kSumChunk ? n - c * kSumChunk : kSumChunk);
      for (int i = 0; i < m; ++i)
        if (sv[buf][i]) {
          sum += st[buf][i];
          ++cnt;
        }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *out_sum = sum;
    *out_cnt = cnt;
  }
}

MetricsWorkspace& metrics_workspace() {
  static std::mutex map_mu;
  static std::map<int, MetricsWorkspace*> per_device;  // never freed: process lifetime
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(map_mu);
  MetricsWorkspace*& w = per_device[dev];
  if (!w) {
    w = new MetricsWorkspace();
    cudaStreamCreateWithFlags(&w->s, cudaStreamNonBlocking);
  }
  return *w;
}

cudaError_t MetricsWorkspace::get(int slot, size_t bytes, void** out) {
  if (bytes + 16 > cap[slot]) {
    if (p[slot]) cudaFree(p[slot]);
    p[slot] = nullptr;
    cap[slot] = 0;
    const size_t want = bytes + bytes / 4 + 16;  // grow with slack
    cudaError_t e = cudaMalloc(&p[slot], want);
    if (e != cudaSuccess) return e;
    cap[slot] = want;
  }
  *out = p[slot];
  return cudaSuccess;
}

#define MET_TRY(x)                    \
  do {                                \
    cudaError_t e_ = (x);             \
    if (e_ != cudaSuccess) return e_; \
  } while (0)

template <typename T>
static cudaError_t ws_get(MetricsWorkspace& ws, int slot, size_t count, T** out) {
  void* q = nullptr;
  cudaError_t e = ws.get(slot, count * sizeof(T), &q);
  *out = static_cast<T*>(q);
  return e;
}

cudaError_t gpu_psnr_parts(MetricsWorkspace& ws, const uchar4* a, const uchar4* b, int n,
                           unsigned long long* sse, unsigned long long* count, cudaStream_t s) {
  unsigned long long* acc;
  MET_TRY(ws_get(ws, MetricsWorkspace::kPsnrAcc, 2, &acc));
  MET_TRY(cudaMemsetAsync(acc, 0, 2 * sizeof(unsigned long long), s));
  const int blocks = std::max(1, std::min(1184, (n + 255) / 256));
  k_psnr_sse<<<blocks, 256, 0, s>>>(a, b, n, acc);
  MET_TRY(cudaGetLastError());
  unsigned long long h[2];
  MET_TRY(cudaMemcpyAsync(h, acc, sizeof(h), cudaMemcpyDeviceToHost, s));
  MET_TRY(cudaStreamSynchronize(s));
  *sse = h[0];
  *count = h[1];
  return cudaSuccess;
}

cudaError_t gpu_ssim_parts(MetricsWorkspace& ws, const uchar4* a, const uchar4* b, int w, int h,
                           double* sum, long long* count, cudaStream_t s) {
  const long long n = static_cast<long long>(w) * h;
  double *tmp, *term, *dsum;
  int* hcnt;
  std::uint8_t* valid;
  MET_TRY(ws_get(ws, MetricsWorkspace::kSsimTmp, static_cast<size_t>(5 * n), &tmp));
  MET_TRY(ws_get(ws, MetricsWorkspace::kSsimTerm, static_cast<size_t>(n), &term));
  MET_TRY(ws_get(ws, MetricsWorkspace::kSsimCnt, static_cast<size_t>(n), &hcnt));
  MET_TRY(ws_get(ws, MetricsWorkspace::kSsimValid, static_cast<size_t>(n), &valid));
  MET_TRY(ws_get(ws, MetricsWorkspace::kSsimSum, 2, &dsum));
  long long* dcnt = reinterpret_cast<long long*>(dsum + 1);
  const SsimKernel g = ssim_kernel();
  const int blocks = static_cast<int>(std::max<long long>(1, std::min<long long>(2368, (n + 255) / 256)));
  k_ssim_h<<<blocks, 256, 0, s>>>(a, b, w, h, g, tmp, hcnt);
  k_ssim_v<<<blocks, 256, 0, s>>>(tmp, hcnt, w, h, g, term, valid);
  k_ssim_sum_staged<<<1, 512, 0, s>>>(term, valid, n, dsum, dcnt);
  MET_TRY(cudaGetLastError());
  MET_TRY(cudaMemcpyAsync(sum, dsum, sizeof(double), cudaMemcpyDeviceToHost, s));
  MET_TRY(cudaMemcpyAsync(count, dcnt, sizeof(long long), cudaMemcpyDeviceToHost, s));
  MET_TRY(cudaStreamSynchronize(s));
  return cudaSuccess;
}

cudaError_t gpu_pack_rgba(MetricsWorkspace& ws, int which, const std::uint8_t* rgb_host,
                          const std::uint8_t* mask_host, int n, uchar4** out, cudaStream_t s) {
  std::uint8_t *drgb, *dmask = nullptr;
  MET_TRY(ws_get(ws, MetricsWorkspace::kPackRgb, static_cast<size_t>(3) * n, &drgb));
  MET_TRY(ws_get(ws, which ? MetricsWorkspace::kPackB : MetricsWorkspace::kPackA,
                 static_cast<size_t>(n), out));
  MET_TRY(cudaMemcpyAsync(drgb, rgb_host, static_cast<size_t>(3) * n, cudaMemcpyHostToDevice, s));
  if (mask_host) {
    MET_TRY(ws_get(ws, MetricsWorkspace::kPackMask, static_cast<size_t>(n), &dmask));
    MET_TRY(cudaMemcpyAsync(dmask, mask_host, static_cast<size_t>(n), cudaMemcpyHostToDevice, s));
  }
  k_pack_rgba<<<std::max(1, std::min(1184, (n + 255) / 256)), 256, 0, s>>>(drgb, dmask, n, *out);
  MET_TRY(cudaGetLastError());
  // the staging buffers are reused by the next pack: order it after this one
  MET_TRY(cudaStreamSynchronize(s));
  return cudaSuccess;
}

}  // namespace stitch_b200_dev
