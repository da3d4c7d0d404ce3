// features_kernels.cu -- feature refinement's image work on the device
// (/root/reference/proj/src/features.cpp:13-234, integral.cpp:8-46): the
// integral image of the quantized gray warped view, the 3-octave x 4-layer
// box-filter Hessian responses over the search region, 3x3x3 non-maximum
// suppression, the keypoint order (one 64-bit radix-sort key per keypoint:
// response descending, then y, x, scale), the upright 64-d descriptors and
// the ratio-test / cross-check matching.  RANSAC over the (hundreds of)
// matches stays in the host layer (refine.cpp), drawing from the
// reference's std::mt19937_64 stream.
//
// Every value follows the reference's arithmetic: u64 box sums, FP64
// responses rounded to float, FP64 Haar statistics with the Gaussian
// weights taken from a host table (libm exp, as the reference), float
// descriptor norms and distances summed in index order, FP64 match
// comparisons -- so keypoints, descriptors and matches equal the oracle's.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "device_math.cuh"
#include "kernels.cuh"

namespace stitch_b200_dev {

constexpr int kFeatOctaves = 3, kFeatLayers = 4;

__host__ __device__ constexpr int feat_filter_size(int octave, int layer) {
  return 3 * ((1 << octave) * (layer + 1) + 1);
}

// ---- integral image (IntegralImage::build, integral.cpp:22-36) ----
// gray = quantize_channel(0.299 r + 0.587 g + 0.114 b) of the warped view
// (invalid pixels are zero RGB, as the reference's warped frame stores them)
__global__ void __launch_bounds__(1024) k_int_rows(const std::uint8_t* __restrict__ rgb, int w,
                                                   int h, unsigned long long* __restrict__ rows) {
  __shared__ unsigned long long sw[32];
  const int y = blockIdx.x;
  const int C = (w + 1023) / 1024;
  const int x0 = threadIdx.x * C;
  unsigned long long loc = 0;
  for (int i = 0; i < C; ++i) {
    const int x = x0 + i;
    if (x >= w) break;
    const std::uint8_t* p = rgb + (static_cast<size_t>(y) * w + x) * 3;
    loc += quantize_d(0.299 * p[0] + 0.587 * p[1] + 0.114 * p[2]);
  }
  // exclusive block scan of the per-thread totals
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long v = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) sw[wid] = v;
  __syncthreads();
  if (wid == 0) {
    unsigned long long t = sw[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long u = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += u;
    }
    sw[lane] = t;
  }
  __syncthreads();
  unsigned long long run = (v - loc) + (wid > 0 ? sw[wid - 1] : 0ull);
  for (int i = 0; i < C; ++i) {
    const int x = x0 + i;
    if (x >= w) break;
    const std::uint8_t* p = rgb + (static_cast<size_t>(y) * w + x) * 3;
    run += quantize_d(0.299 * p[0] + 0.587 * p[1] + 0.114 * p[2]);
    rows[static_cast<size_t>(y) * w + x] = run;
  }
}

// S[(y+1)(w+1) + c] = S[y(w+1) + c] + rowprefix(y, c-1); row 0 and column 0
// are zero (one thread per integral column, rows in order)
__global__ void __launch_bounds__(256) k_int_cols(const unsigned long long* __restrict__ rows,
                                                  int w, int h,
                                                  unsigned long long* __restrict__ S) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > w) return;
  const size_t W = static_cast<size_t>(w) + 1;
  S[c] = 0;
  unsigned long long acc = 0;
  for (int y = 0; y < h; ++y) {
    if (c > 0) acc += rows[static_cast<size_t>(y) * w + c - 1];
    S[(y + 1) * W + c] = acc;
  }
}

struct IntegralView {
  const unsigned long long* s;
  int w, h;
  // box_sum (integral.cpp:38-46)
  __device__ __forceinline__ unsigned long long box(int x0, int y0, int x1, int y1) const {
    x0 = min(max(x0, 0), w);
    x1 = min(max(x1, 0), w);
    y0 = min(max(y0, 0), h);
    y1 = min(max(y1, 0), h);
    if (x1 <= x0 || y1 <= y0) return 0ull;
    const size_t W = static_cast<size_t>(w) + 1;
    return s[y1 * W + x1] - s[y1 * W + x0] - s[y0 * W + x1] + s[y0 * W + x0];
  }
};

// hessian_response (features.cpp:22-44)
__device__ double feat_hessian(const IntegralView& ii, int x, int y, int size) {
  const int lobe = size / 3;
  const int border = (size - 1) / 2;
  const double inv_area = 1.0 / (255.0 * size * size);
  auto box = [&](int bx, int by, int bw, int bh) {
    return static_cast<double>(ii.box(bx, by, bx + bw, by + bh));
  };
  double dxx = box(x - border, y - lobe + 1, size, 2 * lobe - 1) -
               3.0 * box(x - lobe / 2, y - lobe + 1, lobe, 2 * lobe - 1);
  double dyy = box(x - lobe + 1, y - border, 2 * lobe - 1, size) -
               3.0 * box(x - lobe + 1, y - lobe / 2, 2 * lobe - 1, lobe);
  double dxy = box(x + 1, y - lobe, lobe, lobe) + box(x - lobe, y + 1, lobe, lobe) -
               box(x - lobe, y - lobe, lobe, lobe) - box(x + 1, y + 1, lobe, lobe);
  dxx *= inv_area;
  dyy *= inv_area;
  dxy *= inv_area;
  return dxx * dyy - 0.81 * dxy * dxy;
}

// all 12 response layers of the region: layers[(o*4 + l) * rw*rh + y*rw + x]
__global__ void __launch_bounds__(256) k_feat_responses(IntegralView ii, int rx0, int ry0, int rw,
                                                        int rh, float* __restrict__ layers) {
  const long long n = static_cast<long long>(rw) * rh;
  const int ol = blockIdx.y;  // octave-major layer index 0..11
  const int size = feat_filter_size(ol / kFeatLayers + 1, ol % kFeatLayers);
  const int margin = (size - 1) / 2 + 1;
  float* L = layers + ol * n;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int y = static_cast<int>(i / rw), x = static_cast<int>(i - static_cast<long long>(y) * rw);
    const int fx = rx0 + x, fy = ry0 + y;
    float v = 0.0f;
    if (fy >= margin && fy < ii.h - margin && fx >= margin && fx < ii.w - margin)
      v = static_cast<float>(feat_hessian(ii, fx, fy, size));
    L[i] = v;
  }
}

// order-preserving uint of a float (ascending value)
__host__ __device__ __forceinline__ unsigned feat_ord(float f) {
  unsigned b;
#ifdef __CUDA_ARCH__
  b = __float_as_uint(f);
#else
  std::memcpy(&b, &f, 4);
#endif
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// 3x3x3 non-maximum suppression on the interior layers (features.cpp:79-103);
// each keypoint becomes one sort key: ~ord(response) | y | x | scale index.
__global__ void __launch_bounds__(256) k_feat_nms(const float* __restrict__ layers, int rx0,
                                                  int ry0, int rw, int rh, double threshold,
                                                  unsigned long long* __restrict__ keys,
                                                  unsigned* __restrict__ count, unsigned cap) {
  const long long n = static_cast<long long>(rw) * rh;
  const int job = blockIdx.y;  // octave * 2 + (layer - 1)
  const int o = job / 2, l = job % 2 + 1;
  const float* Lm = layers + (o * kFeatLayers + l - 1) * n;
  const float* L0 = Lm + n;
  const float* Lp = L0 + n;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int y = static_cast<int>(i / rw), x = static_cast<int>(i - static_cast<long long>(y) * rw);
    if (y < 1 || y + 1 >= rh || x < 1 || x + 1 >= rw) continue;
    const float v = L0[i];
    if (static_cast<double>(v) <= threshold) continue;
    bool is_max = true;
    for (int dl = -1; dl <= 1 && is_max; ++dl) {
      const float* L = dl < 0 ? Lm : (dl > 0 ? Lp : L0);
      for (int dy = -1; dy <= 1 && is_max; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          if (dl == 0 && dy == 0 && dx == 0) continue;
          if (L[i + static_cast<long long>(dy) * rw + dx] >= v) {
            is_max = false;
            break;
          }
        }
    }
    if (!is_max) continue;
    const unsigned slot = atomicAdd(count, 1u);
    if (slot >= cap) continue;
    const unsigned long long key = (static_cast<unsigned long long>(~feat_ord(v)) << 31) |
                                   (static_cast<unsigned long long>(ry0 + y) << 18) |
                                   (static_cast<unsigned long long>(rx0 + x) << 3) |
                                   static_cast<unsigned long long>(2 * o + (l - 1));
    keys[slot] = key;
  }
}

// the scale of an NMS layer: 1.2 * size / 9 (features.cpp:108)
__host__ __device__ __forceinline__ double feat_scale(int sidx) {
  return 1.2 * feat_filter_size(sidx / 2 + 1, sidx % 2 + 1) / 9.0;
}

struct FeatKeypoint {
  double x, y, scale, response;
};

__global__ void k_feat_decode(const unsigned long long* __restrict__ keys, int n,
                              FeatKeypoint* __restrict__ kps) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long k = keys[i];
  const unsigned ord = ~static_cast<unsigned>(k >> 31);
  const unsigned bits = (ord & 0x80000000u) ? (ord & 0x7fffffffu) : ~ord;
  FeatKeypoint kp;
  kp.x = static_cast<double>((k >> 3) & 0x7fff);
  kp.y = static_cast<double>((k >> 18) & 0x1fff);
  kp.scale = feat_scale(static_cast<int>(k & 7));
  kp.response = static_cast<double>(__uint_as_float(bits));
  kps[i] = kp;
}

// describe (features.cpp:139-179).  gtab[sidx][j20][i20] = the Gaussian
// weight of sample offset ((i20 - 9.5) s, (j20 - 9.5) s), host libm exp.
__global__ void __launch_bounds__(128) k_feat_describe(IntegralView ii,
                                                       const FeatKeypoint* __restrict__ kps, int n,
                                                       const double* __restrict__ gtab,
                                                       float* __restrict__ desc) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const FeatKeypoint kp = kps[k];
  const double s = fmax(1.0, kp.scale);
  int sidx = 0;
  for (int t = 0; t < 6; ++t)
    if (feat_scale(t) == kp.scale) sidx = t;
  const int haar = max(2, static_cast<int>(llround(2.0 * s)));
  const int half = haar / 2;
  float d[64];
  for (int sy = 0; sy < 4; ++sy)
    for (int sx = 0; sx < 4; ++sx) {
      double sdx = 0.0, sdy = 0.0, sadx = 0.0, sady = 0.0;
      for (int j = 0; j < 5; ++j)
        for (int i = 0; i < 5; ++i) {
          const double u = (sx * 5 + i - 9.5) * s;
          const double v = (sy * 5 + j - 9.5) * s;
          const int px = static_cast<int>(llround(kp.x + u));
          const int py = static_cast<int>(llround(kp.y + v));
          const double g = gtab[(sidx * 20 + sy * 5 + j) * 20 + sx * 5 + i];
          const double hx = (static_cast<double>(ii.box(px, py - half, px + half, py + half)) -
                             static_cast<double>(ii.box(px - half, py - half, px, py + half))) /
                            255.0;
          const double hy = (static_cast<double>(ii.box(px - half, py, px + half, py + half)) -
                             static_cast<double>(ii.box(px - half, py - half, px + half, py))) /
                            255.0;
          const double dx = g * hx;
          const double dy = g * hy;
          sdx += dx;
          sdy += dy;
          sadx += fabs(dx);
          sady += fabs(dy);
        }
      const int base = (sy * 4 + sx) * 4;
      d[base + 0] = static_cast<float>(sdx);
      d[base + 1] = static_cast<float>(sdy);
      d[base + 2] = static_cast<float>(sadx);
      d[base + 3] = static_cast<float>(sady);
    }
  float sq = 0.0f;
  for (int i = 0; i < 64; ++i) sq += d[i] * d[i];
  const float norm = sqrtf(sq);
  float* o = desc + 64 * static_cast<size_t>(k);
  for (int i = 0; i < 64; ++i) o[i] = norm > 1e-12f ? d[i] / norm : d[i];
}

// squared descriptor distances, summed in index order in float
__global__ void __launch_bounds__(256) k_feat_dist(const float* __restrict__ da, int na,
                                                   const float* __restrict__ db, int nb,
                                                   float* __restrict__ D) {
  const long long n = static_cast<long long>(na) * nb;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int a = static_cast<int>(t / nb), b = static_cast<int>(t - static_cast<long long>(a) * nb);
    const float* pa = da + 64 * static_cast<size_t>(a);
    const float* pb = db + 64 * static_cast<size_t>(b);
    float sq = 0.0f;
    for (int i = 0; i < 64; ++i) {
      const float e = pa[i] - pb[i];
      sq += e * e;
    }
    D[t] = sq;
  }
}

// match (features.cpp:181-234): per a the nearest / second nearest b and
// the ratio test; per b the nearest a (first a wins ties)
__global__ void k_feat_best_b(const float* __restrict__ D, int na, int nb, double ratio,
                              int* __restrict__ best_b, double* __restrict__ best_dist) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= na) return;
  double d1 = 1.7976931348623157e308, d2 = 1.7976931348623157e308;
  int nearest = -1;
  for (int b = 0; b < nb; ++b) {
    const double d = D[static_cast<size_t>(a) * nb + b];
    if (d < d1) {
      d2 = d1;
      d1 = d;
      nearest = b;
    } else if (d < d2) {
      d2 = d;
    }
  }
  int keep = -1;
  double dist = 0.0;
  if (nearest >= 0 && (nb < 2 || d1 < ratio * ratio * d2)) {
    keep = nearest;
    dist = sqrt(d1);
  }
  best_b[a] = keep;
  best_dist[a] = dist;
}

__global__ void k_feat_best_a(const float* __restrict__ D, int na, int nb,
                              int* __restrict__ best_a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  double best = 1.7976931348623157e308;
  int arg = -1;
  for (int a = 0; a < na; ++a) {
    const double d = D[static_cast<size_t>(a) * nb + b];
    if (d < best) {
      best = d;
      arg = a;
    }
  }
  best_a[b] = arg;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
#define FEAT_TRY(x)                   \
  do {                                \
    cudaError_t e_ = (x);             \
    if (e_ != cudaSuccess) return e_; \
  } while (0)

namespace {
struct Buf {
  void* p = nullptr;
  ~Buf() {
    if (p) cudaFree(p);
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};
}  // namespace

struct FeatView::Impl {
  int w = 0, h = 0;
  Buf integral;
};

FeatView::FeatView() : impl(new Impl) {}
FeatView::~FeatView() { delete impl; }

cudaError_t FeatView::build(const std::uint8_t* d_rgb, int w, int h, cudaStream_t s) {
  impl->w = w;
  impl->h = h;
  Buf rows;
  FEAT_TRY(cudaMalloc(&rows.p, sizeof(unsigned long long) * static_cast<size_t>(w) * h + 16));
  FEAT_TRY(cudaMalloc(&impl->integral.p,
                      sizeof(unsigned long long) * (static_cast<size_t>(w) + 1) * (h + 1)));
  if (w > 1024 * 64) return cudaErrorInvalidValue;
  k_int_rows<<<h, 1024, 0, s>>>(d_rgb, w, h, rows.as<unsigned long long>());
  k_int_cols<<<(w + 1 + 255) / 256, 256, 0, s>>>(rows.as<unsigned long long>(), w, h,
                                                 impl->integral.as<unsigned long long>());
  FEAT_TRY(cudaGetLastError());
  return cudaStreamSynchronize(s);
}

// Gaussian weights of describe(), host libm exactly as features.cpp:162-163
static std::vector<double> gauss_table() {
  std::vector<double> t(6 * 20 * 20);
  for (int sidx = 0; sidx < 6; ++sidx) {
    const double s = std::max(1.0, feat_scale(sidx));
    for (int jj = 0; jj < 20; ++jj)
      for (int ii = 0; ii < 20; ++ii) {
        const double u = (ii - 9.5) * s;
        const double v = (jj - 9.5) * s;
        t[(sidx * 20 + jj) * 20 + ii] = std::exp(-(u * u + v * v) / (2.0 * (3.3 * s) * (3.3 * s)));
      }
  }
  return t;
}

cudaError_t FeatView::detect_describe(int rx0, int ry0, int rx1, int ry1, double threshold,
                                      std::vector<FeatPoint>& kps, std::vector<float>& desc,
                                      cudaStream_t s) const {
  kps.clear();
  desc.clear();
  const int rw = rx1 - rx0, rh = ry1 - ry0;
  const long long n = static_cast<long long>(rw) * rh;
  IntegralView ii{impl->integral.as<unsigned long long>(), impl->w, impl->h};
  Buf layers, keys, keys_sorted, cnt, tmp, dk, dd, dg;
  FEAT_TRY(cudaMalloc(&layers.p, sizeof(float) * 12 * n));
  const unsigned cap = static_cast<unsigned>(6 * n / 9 + 64);
  FEAT_TRY(cudaMalloc(&keys.p, sizeof(unsigned long long) * cap));
  FEAT_TRY(cudaMalloc(&keys_sorted.p, sizeof(unsigned long long) * cap));
  FEAT_TRY(cudaMalloc(&cnt.p, sizeof(unsigned)));
  FEAT_TRY(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned), s));
  const int blocks = static_cast<int>(std::min<long long>(1184, (n + 255) / 256));
  k_feat_responses<<<dim3(blocks, 12), 256, 0, s>>>(ii, rx0, ry0, rw, rh, layers.as<float>());
  k_feat_nms<<<dim3(blocks, 6), 256, 0, s>>>(layers.as<float>(), rx0, ry0, rw, rh, threshold,
                                             keys.as<unsigned long long>(), cnt.as<unsigned>(),
                                             cap);
  FEAT_TRY(cudaGetLastError());
  unsigned count = 0;
  FEAT_TRY(cudaMemcpyAsync(&count, cnt.p, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  FEAT_TRY(cudaStreamSynchronize(s));
  if (count > cap) return cudaErrorInvalidValue;
  if (count == 0) return cudaSuccess;
  size_t tmp_bytes = 0;
  FEAT_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys.as<unsigned long long>(),
                                          keys_sorted.as<unsigned long long>(),
                                          static_cast<int>(count), 0, 64, s));
  FEAT_TRY(cudaMalloc(&tmp.p, tmp_bytes + 16));
  FEAT_TRY(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, keys.as<unsigned long long>(),
                                          keys_sorted.as<unsigned long long>(),
                                          static_cast<int>(count), 0, 64, s));
  FEAT_TRY(cudaMalloc(&dk.p, sizeof(FeatKeypoint) * count));
  k_feat_decode<<<(count + 255) / 256, 256, 0, s>>>(keys_sorted.as<unsigned long long>(),
                                                    static_cast<int>(count),
                                                    dk.as<FeatKeypoint>());
  const std::vector<double> gt = gauss_table();
  FEAT_TRY(cudaMalloc(&dg.p, sizeof(double) * gt.size()));
  FEAT_TRY(cudaMemcpyAsync(dg.p, gt.data(), sizeof(double) * gt.size(), cudaMemcpyHostToDevice, s));
  FEAT_TRY(cudaMalloc(&dd.p, sizeof(float) * 64 * count));
  k_feat_describe<<<(count + 127) / 128, 128, 0, s>>>(ii, dk.as<FeatKeypoint>(),
                                                      static_cast<int>(count), dg.as<double>(),
                                                      dd.as<float>());
  FEAT_TRY(cudaGetLastError());
  std::vector<FeatKeypoint> hk(count);
  desc.resize(static_cast<size_t>(64) * count);
  FEAT_TRY(cudaMemcpyAsync(hk.data(), dk.p, sizeof(FeatKeypoint) * count, cudaMemcpyDeviceToHost, s));
  FEAT_TRY(cudaMemcpyAsync(desc.data(), dd.p, sizeof(float) * desc.size(), cudaMemcpyDeviceToHost, s));
  FEAT_TRY(cudaStreamSynchronize(s));
  kps.resize(count);
  for (unsigned i = 0; i < count; ++i) kps[i] = {hk[i].x, hk[i].y, hk[i].scale, hk[i].response};
  return cudaSuccess;
}

cudaError_t feat_match(const std::vector<float>& da, const std::vector<float>& db, int na, int nb,
                       double ratio, std::vector<int>& best_b, std::vector<double>& best_dist,
                       std::vector<int>& best_a, cudaStream_t s) {
  best_b.assign(na, -1);
  best_dist.assign(na, 0.0);
  best_a.assign(nb, -1);
  if (na == 0 || nb == 0) return cudaSuccess;
  Buf pa, pb, D, bb, bd, ba;
  FEAT_TRY(cudaMalloc(&pa.p, sizeof(float) * da.size()));
  FEAT_TRY(cudaMalloc(&pb.p, sizeof(float) * db.size()));
  FEAT_TRY(cudaMalloc(&D.p, sizeof(float) * static_cast<size_t>(na) * nb));
  FEAT_TRY(cudaMalloc(&bb.p, sizeof(int) * na));
  FEAT_TRY(cudaMalloc(&bd.p, sizeof(double) * na));
  FEAT_TRY(cudaMalloc(&ba.p, sizeof(int) * nb));
  FEAT_TRY(cudaMemcpyAsync(pa.p, da.data(), sizeof(float) * da.size(), cudaMemcpyHostToDevice, s));
  FEAT_TRY(cudaMemcpyAsync(pb.p, db.data(), sizeof(float) * db.size(), cudaMemcpyHostToDevice, s));
  const long long n = static_cast<long long>(na) * nb;
  k_feat_dist<<<static_cast<int>(std::min<long long>(2368, (n + 255) / 256)), 256, 0, s>>>(
      pa.as<float>(), na, pb.as<float>(), nb, D.as<float>());
  k_feat_best_b<<<(na + 127) / 128, 128, 0, s>>>(D.as<float>(), na, nb, ratio, bb.as<int>(),
                                                 bd.as<double>());
  k_feat_best_a<<<(nb + 127) / 128, 128, 0, s>>>(D.as<float>(), na, nb, ba.as<int>());
  FEAT_TRY(cudaGetLastError());
  FEAT_TRY(cudaMemcpyAsync(best_b.data(), bb.p, sizeof(int) * na, cudaMemcpyDeviceToHost, s));
  FEAT_TRY(cudaMemcpyAsync(best_dist.data(), bd.p, sizeof(double) * na, cudaMemcpyDeviceToHost, s));
  FEAT_TRY(cudaMemcpyAsync(best_a.data(), ba.p, sizeof(int) * nb, cudaMemcpyDeviceToHost, s));
  return cudaStreamSynchronize(s);
}

}  // namespace stitch_b200_dev
