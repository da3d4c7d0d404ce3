// geometry_kernels.cu -- init-time pair geometry on the device
// (rebuild_pair_geometry, /root/reference/proj/src/pipeline.cpp:181-205):
// warp masks of every view over the canvas, view footprints, overlap bounds
// (overlap_regions, geometry.cpp:85-117) and the chamfer blend weights
// (blend_weights / chamfer_distance, flow.cpp:192-280).  Used by
// stitch_b200_initialize / stitch_b200_create / stitch_b200_update_geometry,
// so re-refinement (pipeline.cpp:395-406) needs no host pass over the
// canvas.
//
// The chamfer is the reference's two-pass 3-4 raster scan, evaluated
// exactly: a pass is sequential over rows (one CTA per chamfer, rows in
// order), and inside a row the horizontal chain best(x) = min(f(x),
// best(x-1) + 3) is the min-plus prefix scan best(x) = 3x + min_{k<=x}
// (f(k) - 3k) over the row (f = the initial value and the row above's
// +3 / +4 terms).  Distances are integers; the reference's float values are
// exact below 2^24 and saturate at kFarAway = 1e9 (1e9 + 3 rounds to 1e9),
// which the integer form reproduces with a clamp, so the planes are
// bit-identical to the reference's.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "device_math.cuh"
#include "kernels.cuh"

namespace stitch_b200_dev {

constexpr int kChamferInf = 1000000000;  // kFarAway (flow.cpp:14), exact in float
constexpr int kChamferThreads = 1024;
constexpr int kChamferMaxChunk = 64;  // canvas width <= 65536

__device__ __forceinline__ int cadd(int a, int c) { return a >= kChamferInf ? kChamferInf : a + c; }

// extent (bbox) of the valid pixels of masks[view] (& masks[other] when
// other >= 0), plus (views only) a per-column occupancy byte.
// ext: [minx, miny, maxx, maxy] per job, initialised to (w, h, -1, -1).
// *flag = 1 if any byte of the plane is nonzero
__global__ void __launch_bounds__(256) k_plane_any(const std::uint8_t* __restrict__ plane,
                                                   long long n, int* flag) {
  bool on = false;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n && !on;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    on = plane[i] != 0;
  if (__syncthreads_or(on) && threadIdx.x == 0) *flag = 1;
}

__global__ void __launch_bounds__(256) k_mask_extent(const std::uint8_t* __restrict__ masks,
                                                     long long plane, int w, int h,
                                                     const int2* __restrict__ jobs,
                                                     int* __restrict__ ext,
                                                     std::uint8_t* __restrict__ colocc) {
  const int2 jb = jobs[blockIdx.y];
  const std::uint8_t* ma = masks + jb.x * plane;
  const std::uint8_t* mb = jb.y >= 0 ? masks + jb.y * plane : nullptr;
  std::uint8_t* occ = colocc ? colocc + static_cast<long long>(blockIdx.y) * w : nullptr;
  int mnx = w, mny = h, mxx = -1, mxy = -1;
  const long long n = static_cast<long long>(w) * h;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const bool on = ma[i] && (!mb || mb[i]);
    if (!on) continue;
    const int y = static_cast<int>(i / w), x = static_cast<int>(i - static_cast<long long>(y) * w);
    mnx = min(mnx, x);
    mny = min(mny, y);
    mxx = max(mxx, x);
    mxy = max(mxy, y);
    if (occ) occ[x] = 1;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mnx = min(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
    mny = min(mny, __shfl_xor_sync(0xffffffffu, mny, o));
    mxx = max(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
    mxy = max(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
  }
  if ((threadIdx.x & 31) == 0 && mxx >= 0) {
    int* e = ext + 4 * blockIdx.y;
    atomicMin(e + 0, mnx);
    atomicMin(e + 1, mny);
    atomicMax(e + 2, mxx);
    atomicMax(e + 3, mxy);
  }
}

// block-wide exclusive min-scan (forward: over lower thread ids; backward:
// over higher ones) of one int per thread, kChamferThreads threads.
template <bool FWD>
__device__ __forceinline__ int block_excl_min(int v, int* sw) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = FWD ? __shfl_up_sync(0xffffffffu, x, o) : __shfl_down_sync(0xffffffffu, x, o);
    if (FWD ? lane >= o : lane + o < 32) x = min(x, y);
  }
  if (FWD ? lane == 31 : lane == 0) sw[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int t = sw[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = FWD ? __shfl_up_sync(0xffffffffu, t, o) : __shfl_down_sync(0xffffffffu, t, o);
      if (FWD ? lane >= o : lane + o < 32) t = min(t, y);
    }
    sw[32 + lane] = t;  // inclusive over warps
  }
  __syncthreads();
  // exclusive within the block: inclusive-within-warp shifted by one lane,
  // combined with the inclusive total of the preceding (following) warps
  int before = FWD ? __shfl_up_sync(0xffffffffu, x, 1) : __shfl_down_sync(0xffffffffu, x, 1);
  if (FWD ? lane == 0 : lane == 31) before = kChamferInf * 2;
  const int other = FWD ? (wid > 0 ? sw[32 + wid - 1] : kChamferInf * 2)
                        : (wid < 31 ? sw[32 + wid + 1] : kChamferInf * 2);
  const int r = min(before, other);
  __syncthreads();
  return r;
}

// chamfer_distance (flow.cpp:192-223) of zone = masks[a] && !masks[b], one
// CTA per job, both passes in place in D (w*h ints).
__global__ void __launch_bounds__(kChamferThreads) k_chamfer(const std::uint8_t* __restrict__ masks,
                                                             long long plane, int w, int h,
                                                             const int2* __restrict__ jobs,
                                                             int* __restrict__ planes) {
  __shared__ int sw[64];
  const int2 jb = jobs[blockIdx.x];
  const std::uint8_t* ma = masks + jb.x * plane;
  const std::uint8_t* mb = masks + jb.y * plane;
  int* D = planes + blockIdx.x * plane;
  const int C = (w + kChamferThreads - 1) / kChamferThreads;
  const int x0 = threadIdx.x * C;
  int buf[kChamferMaxChunk];
  // forward pass: rows top to bottom, the chain left to right
  for (int y = 0; y < h; ++y) {
    const long long row = static_cast<long long>(y) * w;
    int loc = 2 * kChamferInf;
#pragma unroll 4
    for (int i = 0; i < C; ++i) {
      const int x = x0 + i;
      if (x >= w) break;
      int f = (ma[row + x] && !mb[row + x]) ? 0 : kChamferInf;
      if (y > 0) {
        const int* up = D + row - w;
        f = min(f, cadd(up[x], 3));
        if (x > 0) f = min(f, cadd(up[x - 1], 4));
        if (x + 1 < w) f = min(f, cadd(up[x + 1], 4));
      }
      loc = min(loc, f - 3 * x);
      buf[i] = loc;
    }
    const int carry = block_excl_min<true>(loc, sw);
    for (int i = 0; i < C; ++i) {
      const int x = x0 + i;
      if (x >= w) break;
      D[row + x] = min(kChamferInf, 3 * x + min(carry, buf[i]));
    }
    __syncthreads();
  }
  // backward pass: rows bottom to top, the chain right to left
  for (int y = h - 1; y >= 0; --y) {
    const long long row = static_cast<long long>(y) * w;
    int loc = 2 * kChamferInf;
    for (int i = C - 1; i >= 0; --i) {
      const int x = x0 + i;
      if (x >= w) {
        buf[i] = 2 * kChamferInf;
        continue;
      }
      int f = D[row + x];
      if (y + 1 < h) {
        const int* dn = D + row + w;
        f = min(f, cadd(dn[x], 3));
        if (x + 1 < w) f = min(f, cadd(dn[x + 1], 4));
        if (x > 0) f = min(f, cadd(dn[x - 1], 4));
      }
      loc = min(loc, f + 3 * x);
      buf[i] = loc;
    }
    const int carry = block_excl_min<false>(loc, sw);
    for (int i = 0; i < C; ++i) {
      const int x = x0 + i;
      if (x >= w) break;
      D[row + x] = min(kChamferInf, min(carry, buf[i]) - 3 * x);
    }
    __syncthreads();
  }
}

// blend_weights (flow.cpp:227-280) over one pair's bounds: theta_i from the
// chamfer distances to the exclusive zones of j (to_j) and of i (to_i).
__global__ void __launch_bounds__(256) k_blend_theta(const int* __restrict__ to_j,
                                                     const int* __restrict__ to_i, int w, int bx0,
                                                     int by0, int bw, int bh,
                                                     float* __restrict__ theta) {
  const int n = bw * bh;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int y = i / bw, x = i - y * bw;
    const long long ci_ = static_cast<long long>(by0 + y) * w + bx0 + x;
    const float kFar = 1e9f;
    const float cj = static_cast<float>(to_j[ci_]), ci = static_cast<float>(to_i[ci_]);
    const float di = cj >= kFar ? kFar : fmaxf(0.0f, cj / 3.0f - 1.0f);
    const float dj = ci >= kFar ? kFar : fmaxf(0.0f, ci / 3.0f - 1.0f);
    float ti;
    if (di >= kFar && dj >= kFar)
      ti = 0.5f;
    else if (di >= kFar)
      ti = 1.0f;
    else if (dj >= kFar)
      ti = 0.0f;
    else if (di + dj <= 0.0f)
      ti = 0.5f;
    else
      ti = di / (di + dj);
    theta[i] = ti;
  }
}

#define GEO_TRY(x)                        \
  do {                                    \
    cudaError_t e_ = (x);                 \
    if (e_ != cudaSuccess) return e_;     \
  } while (0)

namespace {
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};
}  // namespace

cudaError_t gpu_init_geometry(const Geometry& geom_in, const double* lift_s, const double* lift_c,
                              const double* lift_h, int n_lift_x, int n_lift_y, int n_views,
                              const std::vector<std::pair<int, int>>& pairs,
                              std::vector<ViewFootprint>& views, std::vector<PairGeometry>& out,
                              const std::vector<const uchar4*>* first_rgba) {
  Geometry geom = geom_in;
  const int w = geom.canvas_w, h = geom.canvas_h;
  const long long P = static_cast<long long>(w) * h;
  cudaStream_t s = nullptr;
  GEO_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg{s};
  DevBuf dlift, dgeom, dmasks, djobs, dext, docc;
  if (geom.projection == 1) {
    const size_t nl = static_cast<size_t>(2 * n_lift_x + n_lift_y);
    GEO_TRY(cudaMalloc(&dlift.p, sizeof(double) * nl));
    double* dl = static_cast<double*>(dlift.p);
    GEO_TRY(cudaMemcpyAsync(dl, lift_s, sizeof(double) * n_lift_x, cudaMemcpyHostToDevice, s));
    GEO_TRY(cudaMemcpyAsync(dl + n_lift_x, lift_c, sizeof(double) * n_lift_x,
                            cudaMemcpyHostToDevice, s));
    GEO_TRY(cudaMemcpyAsync(dl + 2 * n_lift_x, lift_h, sizeof(double) * n_lift_y,
                            cudaMemcpyHostToDevice, s));
    geom.lift_sin = dl;
    geom.lift_cos = dl + n_lift_x;
    geom.lift_h = dl + 2 * n_lift_x;
  }
  GEO_TRY(cudaMalloc(&dgeom.p, sizeof(Geometry)));
  GEO_TRY(cudaMemcpyAsync(dgeom.p, &geom, sizeof(Geometry), cudaMemcpyHostToDevice, s));
  GEO_TRY(cudaMalloc(&dmasks.p, static_cast<size_t>(P) * n_views));
  std::uint8_t* masks = static_cast<std::uint8_t*>(dmasks.p);
  for (int v = 0; v < n_views; ++v)
    launch_warp_mask(static_cast<const Geometry*>(dgeom.p), v, masks + v * P, s);
  GEO_TRY(cudaGetLastError());

  // extents: views (with column occupancy), then pairs (joint masks)
  const int njobs = n_views + static_cast<int>(pairs.size());
  std::vector<int2> jobs(static_cast<size_t>(njobs));
  for (int v = 0; v < n_views; ++v) jobs[v] = make_int2(v, -1);
  for (size_t k = 0; k < pairs.size(); ++k)
    jobs[n_views + k] = make_int2(pairs[k].first, pairs[k].second);
  std::vector<int> ext(static_cast<size_t>(4 * njobs));
  for (int j = 0; j < njobs; ++j) {
    ext[4 * j + 0] = w;
    ext[4 * j + 1] = h;
    ext[4 * j + 2] = -1;
    ext[4 * j + 3] = -1;
  }
  GEO_TRY(cudaMalloc(&djobs.p, sizeof(int2) * njobs));
  GEO_TRY(cudaMalloc(&dext.p, sizeof(int) * ext.size()));
  GEO_TRY(cudaMalloc(&docc.p, static_cast<size_t>(w) * n_views));
  GEO_TRY(cudaMemcpyAsync(djobs.p, jobs.data(), sizeof(int2) * njobs, cudaMemcpyHostToDevice, s));
  GEO_TRY(cudaMemcpyAsync(dext.p, ext.data(), sizeof(int) * ext.size(), cudaMemcpyHostToDevice, s));
  GEO_TRY(cudaMemsetAsync(docc.p, 0, static_cast<size_t>(w) * n_views, s));
  k_mask_extent<<<dim3(296, n_views), 256, 0, s>>>(masks, P, w, h, static_cast<int2*>(djobs.p),
                                                  static_cast<int*>(dext.p),
                                                  static_cast<std::uint8_t*>(docc.p));
  // masked first frames: from here on (pair bounds, chamfer weights) the masks
  // are the warps of those frames (warp_frame with the masked sampler)
  DevBuf dany;
  std::vector<int> any_masked(static_cast<size_t>(n_views), 1);
  if (first_rgba) {
    GEO_TRY(cudaMalloc(&dany.p, sizeof(int) * n_views));
    GEO_TRY(cudaMemsetAsync(dany.p, 0, sizeof(int) * n_views, s));
    for (int v = 0; v < n_views && v < static_cast<int>(first_rgba->size()); ++v)
      if ((*first_rgba)[v]) {
        launch_warp_view(static_cast<const Geometry*>(dgeom.p), v, (*first_rgba)[v], nullptr,
                         masks + v * P, s, true);
        // warp_frame's `any` of the masked first frame (geometry.cpp:79)
        k_plane_any<<<296, 256, 0, s>>>(masks + v * P, P, static_cast<int*>(dany.p) + v);
      }
    GEO_TRY(cudaMemcpyAsync(any_masked.data(), dany.p, sizeof(int) * n_views,
                            cudaMemcpyDeviceToHost, s));
  }
  if (!pairs.empty())
    k_mask_extent<<<dim3(296, static_cast<unsigned>(pairs.size())), 256, 0, s>>>(
        masks, P, w, h, static_cast<int2*>(djobs.p) + n_views,
        static_cast<int*>(dext.p) + 4 * n_views, nullptr);
  GEO_TRY(cudaGetLastError());
  std::vector<std::uint8_t> occ(static_cast<size_t>(w) * n_views);
  GEO_TRY(cudaMemcpyAsync(ext.data(), dext.p, sizeof(int) * ext.size(), cudaMemcpyDeviceToHost, s));
  GEO_TRY(cudaMemcpyAsync(occ.data(), docc.p, occ.size(), cudaMemcpyDeviceToHost, s));
  GEO_TRY(cudaStreamSynchronize(s));
  views.assign(static_cast<size_t>(n_views), ViewFootprint{});
  for (int v = 0; v < n_views; ++v) {
    ViewFootprint& f = views[v];
    f.masked_empty = first_rgba && v < static_cast<int>(first_rgba->size()) &&
                     (*first_rgba)[v] && any_masked[v] == 0;
    f.empty = ext[4 * v + 2] < 0;
    if (f.empty) continue;
    f.bbox[0] = ext[4 * v + 0];
    f.bbox[1] = ext[4 * v + 1];
    f.bbox[2] = ext[4 * v + 2] + 1;
    f.bbox[3] = ext[4 * v + 3] + 1;
    // widest run of empty columns inside the bbox (wrapped ring views)
    const std::uint8_t* col = occ.data() + static_cast<size_t>(v) * w;
    f.gap[0] = f.gap[1] = 0;
    int best = 0;
    for (int x = f.bbox[0]; x < f.bbox[2];) {
      if (col[x]) {
        ++x;
        continue;
      }
      int e = x;
      while (e < f.bbox[2] && !col[e]) ++e;
      if (e - x > best) {
        best = e - x;
        f.gap[0] = x;
        f.gap[1] = e;
      }
      x = e;
    }
  }
  out.assign(pairs.size(), PairGeometry{});
  if (pairs.empty()) return cudaSuccess;
  for (size_t k = 0; k < pairs.size(); ++k) {
    const int* e = ext.data() + 4 * (n_views + k);
    PairGeometry& pg = out[k];
    pg.ok = e[2] >= 0;
    if (!pg.ok) continue;
    pg.bounds[0] = e[0];
    pg.bounds[1] = e[1];
    pg.bounds[2] = e[2] + 1;
    pg.bounds[3] = e[3] + 1;
  }
  if (w > kChamferThreads * kChamferMaxChunk) return cudaErrorInvalidValue;
  // chamfer planes: jobs (view, partner) -> to_i, (partner, view) -> to_j;
  // processed in groups bounded to ~4 GiB of planes (init-time scratch)
  const long long per_pair = 2 * P * static_cast<long long>(sizeof(int));
  const int group = static_cast<int>(std::max<long long>(1, (4ll << 30) / per_pair));
  DevBuf dplanes, dcj, dtheta;
  const int gsz = std::min<int>(group, static_cast<int>(pairs.size()));
  GEO_TRY(cudaMalloc(&dplanes.p, static_cast<size_t>(per_pair) * gsz));
  GEO_TRY(cudaMalloc(&dcj.p, sizeof(int2) * 2 * gsz));
  size_t max_theta = 16;
  for (const PairGeometry& pg : out)
    if (pg.ok)
      max_theta = std::max(max_theta, static_cast<size_t>(pg.bounds[2] - pg.bounds[0]) *
                                          (pg.bounds[3] - pg.bounds[1]));
  GEO_TRY(cudaMalloc(&dtheta.p, sizeof(float) * max_theta));
  int* planes = static_cast<int*>(dplanes.p);
  for (size_t k0 = 0; k0 < pairs.size(); k0 += gsz) {
    const size_t k1 = std::min(pairs.size(), k0 + gsz);
    std::vector<int2> cj;
    for (size_t k = k0; k < k1; ++k) {
      cj.push_back(make_int2(pairs[k].first, pairs[k].second));   // zone_i -> to_i
      cj.push_back(make_int2(pairs[k].second, pairs[k].first));   // zone_j -> to_j
    }
    GEO_TRY(cudaMemcpyAsync(dcj.p, cj.data(), sizeof(int2) * cj.size(), cudaMemcpyHostToDevice, s));
    k_chamfer<<<static_cast<unsigned>(cj.size()), kChamferThreads, 0, s>>>(
        masks, P, w, h, static_cast<int2*>(dcj.p), planes);
    GEO_TRY(cudaGetLastError());
    for (size_t k = k0; k < k1; ++k) {
      PairGeometry& pg = out[k];
      if (!pg.ok) continue;
      const int* to_i = planes + 2 * (k - k0) * P;
      const int* to_j = to_i + P;
      const int bw = pg.bounds[2] - pg.bounds[0], bh = pg.bounds[3] - pg.bounds[1];
      const int n = bw * bh;
      k_blend_theta<<<std::max(1, std::min(1184, (n + 255) / 256)), 256, 0, s>>>(
          to_j, to_i, w, pg.bounds[0], pg.bounds[1], bw, bh, static_cast<float*>(dtheta.p));
      GEO_TRY(cudaGetLastError());
      pg.theta.resize(static_cast<size_t>(n));
      GEO_TRY(cudaMemcpyAsync(pg.theta.data(), dtheta.p, sizeof(float) * n, cudaMemcpyDeviceToHost,
                              s));
      GEO_TRY(cudaStreamSynchronize(s));
    }
  }
  return cudaSuccess;
}

}  // namespace stitch_b200_dev
