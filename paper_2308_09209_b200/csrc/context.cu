// context.cu -- the C ABI (include/stitch_b200.h): device contexts, the
// per-frame launch plan captured once as a CUDA graph, uploads/downloads,
// and the standalone initialize() (pipeline.cpp:209-257, refinement off).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <cstring>
#include <memory>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "host_geometry.hpp"
#include "kernels.cuh"
#include "stitch_b200.h"

using namespace stitch_b200_dev;
namespace hg_ns = stitch_b200_host;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      return fail(STITCH_B200_CudaError, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

enum OpKind { OP_EXPAND, OP_CROP, OP_STATS, OP_SOLVE, OP_PREP, OP_PYR, OP_HSPREP, OP_HS, OP_CANVAS,
              OP_BALANCE, OP_TONE, OP_EVENT };

struct Op {
  OpKind kind;
  int offset = 0, count = 0;  // task table slice or pair list slice
  int max_w = 0, max_h = 0, max_px = 0;
  int event = 0;
  int sweeps = 0;  // OP_HS: Jacobi sweeps of this launch (segment length)
  int fuse = 0;    // OP_HS: 1 also linearises this warp iteration (prologue),
                   // 2 also the next one (epilogue)
};

}  // namespace

// One pipeline slot: the buffers a frame writes (RGBA views, crops,
// pyramids, flows, panorama), its device geometry / frame state / task
// tables, its compute stream and its graphs.  Two slots let consecutive
// frames overlap; the temporal state is shared and updated in frame order.
struct SlotRes {
  Geometry hg{};           // host mirror (this slot's buffer pointers)
  Geometry* dg = nullptr;  // device geometry
  DevState* dst = nullptr;
  uchar4* d_pano = nullptr;
  CanvasParams cparams{};
  HsTask* d_hs = nullptr;
  PrepTask* d_hp = nullptr;
  PyrTask* d_pyr = nullptr;
  cudaStream_t cs = nullptr;
  // the frame as 4 graphs: front (expand, crops), colour (3D-M solves, in
  // frame order across slots), mid (flow), back (canvas + balance, in frame
  // order across slots; tone)
  static constexpr int kSegs = 4;
  cudaGraph_t graph[kSegs] = {};
  cudaGraphExec_t exec[kSegs] = {};
};

// Host copy pool for the pageable-buffer path.  The reference hands frames
// over as pageable std::vector buffers (frame.hpp:17-57, pipeline.hpp:65-80);
// an async copy from pageable memory would serialise the pipeline (the
// driver stages it synchronously, and a D2H to pageable memory returns only
// after the copy), so such buffers go through a pinned per-slot ring and
// these workers move the bytes between the caller's buffers and the ring in
// parallel chunks while the GPU works on the other frames in flight.
class CopyPool {
 public:
  struct Job {
    void* dst;
    const void* src;
    size_t n;
  };

  explicit CopyPool(int workers) {
    for (int i = 0; i < workers; ++i) th_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }

  // Copies every (dst, src, n), split into ~1 MiB chunks; the calling thread
  // works too.  Returns when all bytes have landed.  Each call is its own
  // batch, shared with the workers that join it, so a worker that wakes late
  // can only ever claim chunks of a batch it holds alive.
  void run(const std::vector<Job>& jobs) {
    constexpr size_t kChunk = size_t(1) << 20;
    auto b = std::make_shared<Batch>();
    for (const Job& j : jobs)
      for (size_t o = 0; o < j.n; o += kChunk)
        b->chunks.push_back({static_cast<char*>(j.dst) + o, static_cast<const char*>(j.src) + o,
                             std::min(kChunk, j.n - o)});
    if (b->chunks.empty()) return;
    if (b->chunks.size() == 1 || th_.empty()) {  // small: no hand-off
      for (const Job& c : b->chunks) std::memcpy(c.dst, c.src, c.n);
      return;
    }
    b->left = b->chunks.size();
    {
      std::lock_guard<std::mutex> lk(mu_);
      batch_ = b;
      ++gen_;
    }
    cv_.notify_all();
    drain(*b);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return b->left == 0; });
    if (batch_ == b) batch_.reset();
  }

 private:
  struct Batch {
    std::vector<Job> chunks;
    std::atomic<size_t> next{0};
    size_t left = 0;  // guarded by mu_
  };

  void drain(Batch& b) {
    size_t did = 0;
    for (size_t i = b.next.fetch_add(1); i < b.chunks.size(); i = b.next.fetch_add(1)) {
      std::memcpy(b.chunks[i].dst, b.chunks[i].src, b.chunks[i].n);
      ++did;
    }
    if (did) {
      std::lock_guard<std::mutex> lk(mu_);
      b.left -= did;
      if (b.left == 0) done_cv_.notify_all();
    }
  }

  void loop() {
    unsigned long long seen = 0;
    for (;;) {
      std::shared_ptr<Batch> b;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        b = batch_;
      }
      if (b) drain(*b);
    }
  }

  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::shared_ptr<Batch> batch_;
  unsigned long long gen_ = 0;
  bool stop_ = false;
};

// Only plain pageable host memory is staged.  Page-locked (cudaHostAlloc'ed or
// cudaHostRegister'ed) memory is the direct source / target of an async copy,
// and so is anything else the runtime knows (device or managed memory: the
// copy then fails or succeeds on the runtime's terms, but the host never
// dereferences a device address).
bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type != cudaMemoryTypeUnregistered;
}

struct Ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;  // the API stream (process_device, profile, debug)
  // pipeline slots: frames in flight (STITCH_B200_SLOTS, 2..kMaxSlots;
  // default 4), fixed when the context is built
  static constexpr int kMaxSlots = 8;
  int n_slots = 4;
  SlotRes slot[kMaxSlots];
  Geometry hg{};  // metadata (slot 0's mirror; buffers: use slot[s].hg)
  TemporalState* dtemp = nullptr;
  stitch_b200_init init{};  // copy (theta pointers re-pointed at host copies)
  std::vector<std::vector<float>> theta_host;
  std::vector<int> refine_warning;  // per pair (initialize_frames with refinement)
  std::vector<void*> allocs;
  std::uint8_t* d_frames[kMaxViews] = {};
  size_t frame_bytes[kMaxViews] = {};
  // per slot: inputs, outputs, stage events, report
  std::uint8_t* d_in[kMaxSlots][kMaxViews] = {};
  std::uint8_t* d_out_rgb[kMaxSlots] = {};
  std::uint8_t* d_out_mask[kMaxSlots] = {};
  long long n_px = 0;
  int max_crop_px = 0;
  int max_crop_w = 0, max_crop_h = 0;
  long long max_view_px = 0;
  int sweeps = 10;
  float alpha2 = 225.0f;
  int n_levels_max = 0;
  std::vector<Op> plan;
  int seg_begin[SlotRes::kSegs + 1] = {};  // plan index ranges of the segments
  int* d_lists = nullptr;
  int launches = 0;
  cudaEvent_t ev[kMaxSlots][6] = {};
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t h2d_done[kMaxSlots] = {}, comp_done[kMaxSlots] = {}, d2h_done[kMaxSlots] = {};
  // frame-order points between slots: colour solves done, canvas done
  cudaEvent_t color_done[kMaxSlots] = {}, canvas_done[kMaxSlots] = {};
  cudaEvent_t fork_ev = nullptr;
  long long seq = 0;                       // frames submitted (any API)
  long long slot_ticket[kMaxSlots];  // ticket occupying each slot
  bool slot_pending[kMaxSlots];
  bool slot_joined[kMaxSlots];  // the API stream waited for the slot's frame
  std::vector<std::pair<long long, stitch_b200_report>> done_reports;
  int last_slot = 0;
  // pinned ring for device-frame pointer tables
  FrameTable* h_ptr_ring = nullptr;  // pinned ring of per-frame tables
  cudaEvent_t ring_ev[16] = {};
  int ring_pos = 0;
  DevReport* h_report = nullptr;  // one per slot (pinned)
  // pageable caller buffers: pinned staging per slot (allocated on first
  // use), the caller's output pointers to fill when the slot retires, and
  // the copy workers
  std::uint8_t* h_stage_in[kMaxSlots][kMaxViews] = {};
  // input masks (Frame::mask) of host-path frames: device buffers per slot
  // (allocated on the first masked frame) and their pinned staging
  std::uint8_t* d_mask[kMaxSlots][kMaxViews] = {};
  std::uint8_t* h_stage_min[kMaxSlots][kMaxViews] = {};
  std::uint8_t* h_stage_rgb[kMaxSlots] = {};
  std::uint8_t* h_stage_mask[kMaxSlots] = {};
  std::uint8_t* user_rgb[kMaxSlots] = {};
  std::uint8_t* user_mask[kMaxSlots] = {};
  // staged outputs leave the device in chunks, each followed by an event, so
  // the copy of chunk c into the caller's buffer overlaps the DMA of c + 1
  static constexpr int kOutChunks = 16;
  struct OutChunk {
    std::uint8_t* dst;
    const std::uint8_t* src;
    size_t n;
  };
  std::vector<OutChunk> out_chunks[kMaxSlots];
  cudaEvent_t out_ev[kMaxSlots][kOutChunks] = {};
  std::unique_ptr<CopyPool> copier;
  // coverage of masked frames (EmptyProjection): device word + pinned copy
  unsigned* d_cover = nullptr;
  unsigned* h_cover = nullptr;
  std::vector<int> pair_levels;
  float2* d_zero = nullptr;

  Ctx() {
    for (int s = 0; s < kMaxSlots; ++s) {
      slot_ticket[s] = -1;
      slot_pending[s] = false;
      slot_joined[s] = true;
    }
  }

  ~Ctx() {
    if (stream) cudaStreamSynchronize(stream);
    for (auto& S : slot)
      if (S.cs) cudaStreamSynchronize(S.cs);
    if (h2d) cudaStreamSynchronize(h2d);
    if (d2h) cudaStreamSynchronize(d2h);
    for (int s = 0; s < kMaxSlots; ++s) {
      for (int g = 0; g < SlotRes::kSegs; ++g) {
        if (slot[s].exec[g]) cudaGraphExecDestroy(slot[s].exec[g]);
        if (slot[s].graph[g]) cudaGraphDestroy(slot[s].graph[g]);
      }
      for (auto& e : ev[s])
        if (e) cudaEventDestroy(e);
      for (cudaEvent_t e : {h2d_done[s], comp_done[s], d2h_done[s], color_done[s], canvas_done[s]})
        if (e) cudaEventDestroy(e);
      if (slot[s].cs) cudaStreamDestroy(slot[s].cs);
    }
    if (fork_ev) cudaEventDestroy(fork_ev);
    if (h2d) cudaStreamDestroy(h2d);
    if (d2h) cudaStreamDestroy(d2h);
    for (auto& e : ring_ev)
      if (e) cudaEventDestroy(e);
    for (void* p : allocs) cudaFree(p);
    if (h_ptr_ring) cudaFreeHost(h_ptr_ring);
    if (h_report) cudaFreeHost(h_report);
    if (h_cover) cudaFreeHost(h_cover);
    for (int s = 0; s < kMaxSlots; ++s) {
      for (auto* q : h_stage_in[s])
        if (q) cudaFreeHost(q);
      for (auto* q : h_stage_min[s])
        if (q) cudaFreeHost(q);
      if (h_stage_rgb[s]) cudaFreeHost(h_stage_rgb[s]);
      for (cudaEvent_t e : out_ev[s])
        if (e) cudaEventDestroy(e);
      if (h_stage_mask[s]) cudaFreeHost(h_stage_mask[s]);
    }
    if (stream) cudaStreamDestroy(stream);
  }

  template <typename T>
  cudaError_t alloc(T** p, size_t count) {
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, std::max<size_t>(count * sizeof(T), 16));
    if (e != cudaSuccess) return e;
    allocs.push_back(q);
    *p = static_cast<T*>(q);
    return cudaMemset(q, 0, std::max<size_t>(count * sizeof(T), 16));
  }
};

struct stitch_b200_ctx {
  std::unique_ptr<Ctx> c;
};

namespace {

int validate_init(const stitch_b200_init* in) {
  if (in->n_views < 2 || in->n_views > kMaxViews)
    return fail(STITCH_B200_ConfigurationError, "n_views must be in [2, 16]");
  if (in->reference < 0 || in->reference >= in->n_views)
    return fail(STITCH_B200_ConfigurationError, "reference view index out of range");
  if (in->canvas_width <= 0 || in->canvas_height <= 0)
    return fail(STITCH_B200_ConfigurationError, "empty canvas");
  if (in->n_pairs < 0 || in->n_pairs > kMaxPairs)
    return fail(STITCH_B200_ConfigurationError, "too many pairs");
  for (int v = 0; v < in->n_views; ++v)
    if (in->view_width[v] <= 0 || in->view_height[v] <= 0)
      return fail(STITCH_B200_ConfigurationError, "view size must be positive");
  if (!(in->lambda > 0.0 && in->lambda < 0.5))
    return fail(STITCH_B200_ConfigError, "balance.lambda must be in (0, 0.5)");
  if (in->flow_levels < 1 || in->flow_iterations < 1 || !(in->smoothness > 0.0))
    return fail(STITCH_B200_ConfigError, "flow levels/iterations/smoothness must be positive");
  for (int k = 0; k < in->n_pairs; ++k) {
    const stitch_b200_pair& p = in->pairs[k];
    if (p.view < 0 || p.view >= in->n_views || p.partner < 0 || p.partner >= in->n_views ||
        p.view == p.partner || p.view == in->reference)
      return fail(STITCH_B200_ConfigurationError, "bad pair views");
    if (p.x1 <= p.x0 || p.y1 <= p.y0 || p.x0 < 0 || p.y0 < 0 || p.x1 > in->canvas_width ||
        p.y1 > in->canvas_height)
      return fail(STITCH_B200_EmptyRegion, "pair bounds outside the canvas");
    if (!p.theta_i) return fail(STITCH_B200_MissingState, "pair weights missing");
  }
  // a partner must be the reference or a view corrected by an earlier pair
  for (int k = 0; k < in->n_pairs; ++k) {
    const int partner = in->pairs[k].partner;
    if (partner == in->reference) continue;
    bool found = false;
    for (int j = 0; j < k; ++j)
      if (in->pairs[j].view == partner) found = true;
    if (!found)
      return fail(STITCH_B200_ConfigurationError,
                  "pair partner must be the reference or corrected by an earlier pair");
  }
  return STITCH_B200_OK;
}

// Lift tables of the cylindrical canvas (extension); empty for planar.
struct LiftTables {
  std::vector<double> s, c, h;
};

LiftTables make_lift(const stitch_b200_init* in) {
  LiftTables t;
  if (in->projection == 1) {
    hg_ns::Canvas cv;
    cv.width = in->canvas_width;
    cv.height = in->canvas_height;
    cv.offx = in->canvas_offset[0];
    cv.offy = in->canvas_offset[1];
    hg_ns::lift_tables(cv, in->cyl_focal, t.s, t.c, t.h);
  }
  return t;
}

// Init geometry on the device (geometry_kernels.cu): view footprints and,
// for the given pairs, overlap bounds + blend weights.
int init_geometry(int device, const Geometry& geom, const LiftTables& lt, int n_views,
                  const std::vector<std::pair<int, int>>& pairs, std::vector<ViewFootprint>& views,
                  std::vector<PairGeometry>& pair_geo,
                  const std::vector<const uchar4*>* first_rgba = nullptr) {
  CUDA_TRY(cudaSetDevice(device));
  CUDA_TRY(gpu_init_geometry(geom, lt.s.data(), lt.c.data(), lt.h.data(),
                             static_cast<int>(lt.s.size()), static_cast<int>(lt.h.size()), n_views,
                             pairs, views, pair_geo, first_rgba));
  return STITCH_B200_OK;
}

void fill_views(Geometry& g, const stitch_b200_init* in) {
  g.projection = in->projection == 1 ? 1 : 0;
  g.canvas_w = in->canvas_width;
  g.canvas_h = in->canvas_height;
  g.offx = in->canvas_offset[0];
  g.offy = in->canvas_offset[1];
  g.n_views = in->n_views;
  g.reference = in->reference;
  for (int v = 0; v < in->n_views; ++v) {
    g.views[v].width = in->view_width[v];
    g.views[v].height = in->view_height[v];
    for (int i = 0; i < 9; ++i) g.views[v].inv[i] = in->inv_maps[v][i];
  }
}

int enqueue_op(Ctx* ctx, const Op& op, cudaStream_t s, int slot = 0) {
  const Geometry& g = ctx->hg;
  const SlotRes& S = ctx->slot[slot];
  switch (op.kind) {
    case OP_EXPAND:
      launch_expand(S.dg, g.n_views, ctx->max_view_px, s);
      return 1;
    case OP_CROP:
      if (!g.n_pairs) return 0;
      launch_crop_warp(S.cparams, ctx->max_crop_w, ctx->max_crop_h, s);
      return 1;
    case OP_STATS:
      return launch_pair_color(S.dg, S.dst, ctx->d_lists + op.offset, op.count, ctx->max_crop_px,
                               s);
    case OP_PREP:
      if (!g.n_pairs) return 0;
      if (op.fuse)
        launch_flow_prepare_pyr(S.dg, S.dst, g.n_pairs, ctx->max_crop_w, ctx->max_crop_h, s);
      else
        launch_flow_prepare(S.dg, S.dst, g.n_pairs, ctx->max_crop_px, s);
      return 1;
    case OP_PYR:
      launch_pyr_down(S.d_pyr + op.offset, op.count, op.max_px, s);
      return 1;
    case OP_HSPREP:
      launch_hs_prepare(S.d_hp + op.offset, op.count, op.max_w, op.max_h, ctx->alpha2, s);
      return 1;
    case OP_HS:
      launch_hs_iter(S.d_hs + op.offset, op.count, op.max_w, op.max_h, op.sweeps, op.fuse,
                     ctx->alpha2, s);
      return 1;
    case OP_CANVAS:
      return launch_canvas(S.cparams, S.dg, S.dst, S.d_pano, ctx->num_sms, s);
    case OP_TONE:
      launch_tone(S.dst, S.d_pano, ctx->n_px, ctx->d_out_rgb[slot], ctx->d_out_mask[slot], s);
      return 1;
    default:
      return 0;
  }
}

int build_context(const stitch_b200_init* in, int device,
                  const std::vector<ViewFootprint>* views_in, std::unique_ptr<Ctx>& out) {
  int rc = validate_init(in);
  if (rc) return rc;
  auto ctx = std::make_unique<Ctx>();
  ctx->device = device;
  {
    static const int slots = env_int("STITCH_B200_SLOTS", 4);
    ctx->n_slots = std::min(Ctx::kMaxSlots, std::max(2, slots));
  }
  CUDA_TRY(cudaSetDevice(device));
  CUDA_TRY(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
  CUDA_TRY(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  ctx->init = *in;
  Geometry& g = ctx->hg;
  std::memset(&g, 0, sizeof(g));
  fill_views(g, in);
  g.n_pairs = in->n_pairs;
  g.weighting = in->fuse_weighting ? 1 : 0;
  g.lambda = in->lambda;
  g.gamma_dark = in->gamma_dark;
  g.gamma_bright = in->gamma_bright;
  g.target_black = in->target_black;
  g.target_white = in->target_white;
  g.curve_ok = (in->gamma_dark > 0.0 && in->gamma_bright > 0.0 &&
                in->target_black <= in->target_white)
                   ? 1
                   : 0;

  // view footprints (bbox of the warp mask); EmptyProjection if none.
  std::vector<ViewFootprint> views_local;
  const std::vector<ViewFootprint>* views = views_in;
  const LiftTables lift = make_lift(in);
  if (g.projection == 1) {
    if (!(in->cyl_focal > 0.0) ||
        static_cast<size_t>(in->canvas_width) != lift.s.size())
      return fail(STITCH_B200_ConfigurationError, "cylindrical canvas needs cyl_focal > 0");
    double* dl;
    CUDA_TRY(ctx->alloc(&dl, lift.s.size() + lift.c.size() + lift.h.size()));
    CUDA_TRY(cudaMemcpy(dl, lift.s.data(), sizeof(double) * lift.s.size(), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(dl + lift.s.size(), lift.c.data(), sizeof(double) * lift.c.size(),
                        cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(dl + lift.s.size() + lift.c.size(), lift.h.data(),
                        sizeof(double) * lift.h.size(), cudaMemcpyHostToDevice));
    g.lift_sin = dl;
    g.lift_cos = dl + lift.s.size();
    g.lift_h = dl + lift.s.size() + lift.c.size();
  }
  if (!views) {
    std::vector<PairGeometry> none;
    rc = init_geometry(device, g, lift, in->n_views, {}, views_local, none);
    if (rc) return rc;
    views = &views_local;
  }
  for (int v = 0; v < in->n_views; ++v) {
    const ViewFootprint& f = (*views)[v];
    if (f.empty) return fail(STITCH_B200_EmptyProjection, "a view projects to no canvas pixel");
    for (int i = 0; i < 4; ++i) g.views[v].bbox[i] = f.bbox[i];
    g.views[v].gap[0] = f.gap[0];
    g.views[v].gap[1] = f.gap[1];
  }

  // ---- per-slot buffers, geometry and task tables (the plan is identical
  // for every slot; the temporal state is shared) ----
  CUDA_TRY(ctx->alloc(&ctx->dtemp, 1));
  {
    // window capacity (TransferWindow clamps to 1..3, color_transfer.cpp:8-11)
    std::unique_ptr<TemporalState> ts(new TemporalState());
    std::memset(ts.get(), 0, sizeof(TemporalState));
    const int cap = std::min(3, std::max(1, in->window_capacity));
    for (int k = 0; k < kMaxPairs; ++k) ts->windows[k].capacity = cap;
    CUDA_TRY(cudaMemcpy(ctx->dtemp, ts.get(), sizeof(TemporalState), cudaMemcpyHostToDevice));
  }
  const Geometry base = g;
  std::vector<float*> theta_dev(in->n_pairs, nullptr);
  for (int sl = 0; sl < ctx->n_slots; ++sl) {
    SlotRes& S = ctx->slot[sl];
    Geometry& g = S.hg;
    g = base;
    // buffers
    for (int v = 0; v < in->n_views; ++v) {
      ctx->frame_bytes[v] = static_cast<size_t>(in->view_width[v]) * in->view_height[v] * 3;
      if (sl == 0) {
        CUDA_TRY(ctx->alloc(&ctx->d_frames[v], ctx->frame_bytes[v]));
        ctx->d_in[0][v] = ctx->d_frames[v];
        for (int s2 = 1; s2 < ctx->n_slots; ++s2)
          CUDA_TRY(ctx->alloc(&ctx->d_in[s2][v], ctx->frame_bytes[v]));
      }
      g.in.frames[v] = ctx->d_in[sl][v];
      const long long vpx = static_cast<long long>(in->view_width[v]) * in->view_height[v];
      CUDA_TRY(ctx->alloc(&g.rgba[v], vpx));
      ctx->max_view_px = std::max(ctx->max_view_px, vpx);
    }
    ctx->n_px = static_cast<long long>(g.canvas_w) * g.canvas_h;
    CUDA_TRY(ctx->alloc(&S.d_pano, static_cast<size_t>(ctx->n_px) + 4));
    CUDA_TRY(ctx->alloc(&ctx->d_out_rgb[sl], static_cast<size_t>(ctx->n_px) * 3 + 16));
    CUDA_TRY(ctx->alloc(&ctx->d_out_mask[sl], static_cast<size_t>(ctx->n_px) + 16));

    ctx->sweeps = std::max(1, in->flow_iterations / 5);  // flow.cpp:79-80
    ctx->alpha2 = static_cast<float>(in->smoothness * in->smoothness);
    ctx->theta_host.resize(in->n_pairs);
    int max_zero = 16;
    for (int k = 0; k < in->n_pairs; ++k) {
      const stitch_b200_pair& sp = in->pairs[k];
      PairDesc& p = g.pairs[k];
      p.view = sp.view;
      p.partner = sp.partner;
      p.x0 = sp.x0;
      p.y0 = sp.y0;
      p.w = sp.x1 - sp.x0;
      p.h = sp.y1 - sp.y0;
      const int n = p.w * p.h;
      ctx->max_crop_px = std::max(ctx->max_crop_px, n);
      ctx->max_crop_w = std::max(ctx->max_crop_w, p.w);
      ctx->max_crop_h = std::max(ctx->max_crop_h, p.h);
      max_zero = std::max(max_zero, n);
      ctx->theta_host[k].assign(sp.theta_i, sp.theta_i + n);
      ctx->init.pairs[k].theta_i = ctx->theta_host[k].data();
      if (!theta_dev[k]) {  // constant: shared by the slots
        CUDA_TRY(ctx->alloc(&theta_dev[k], n));
        CUDA_TRY(cudaMemcpy(theta_dev[k], sp.theta_i, sizeof(float) * n, cudaMemcpyHostToDevice));
      }
      p.theta_i = theta_dev[k];
      for (int s = 0; s < 2; ++s) {
        CUDA_TRY(ctx->alloc(&p.crop_raw[s], n));
        CUDA_TRY(ctx->alloc(&p.crop_cor[s], n));
      }
      // dense_flow requires >= 16x16 (flow.cpp:146-148), else zero flow
      p.flow_ok = (p.w >= 16 && p.h >= 16) ? 1 : 0;
    }
    if (sl == 0) CUDA_TRY(ctx->alloc(&ctx->d_zero, max_zero));

    // pair depth (distance from the reference through partners)
    std::vector<int> depth(in->n_pairs, 1);
    int max_depth = 0;
    for (int k = 0; k < in->n_pairs; ++k) {
      const int partner = in->pairs[k].partner;
      if (partner != in->reference)
        for (int j = 0; j < k; ++j)
          if (in->pairs[j].view == partner) depth[k] = depth[j] + 1;
      g.pair_depth[k] = depth[k];
      max_depth = std::max(max_depth, depth[k]);
    }

    // ---- flow plan: pyramids (flow.cpp:152-156), per-level tasks ----
    struct TaskState {
      int k, dir, L;
      int dims[kMaxLevels][2];
      float2* UV[2];  // (u, v) ping-pong
      float4* KQ[2];  // (gx, gy, c, denom) per pixel: current warp iteration /
                      // the next one's, written by an epilogue linearisation
      int cur, kc;
    };
    std::vector<TaskState> tasks;
    ctx->pair_levels.assign(in->n_pairs, 0);
    int Lmax = 0;
    for (int k = 0; k < in->n_pairs; ++k) {
      PairDesc& p = g.pairs[k];
      if (!p.flow_ok) {
        for (int d = 0; d < 2; ++d) {
          p.flow_uv[d] = ctx->d_zero;
        }
        continue;
      }
      int dims[kMaxLevels][2];
      int L = 1;
      dims[0][0] = p.w;
      dims[0][1] = p.h;
      for (int l = 1; l < in->flow_levels && l < kMaxLevels; ++l) {
        if (dims[l - 1][0] < 16 || dims[l - 1][1] < 16) break;
        dims[l][0] = std::max(1, dims[l - 1][0] / 2);
        dims[l][1] = std::max(1, dims[l - 1][1] / 2);
        ++L;
      }
      ctx->pair_levels[k] = L;
      Lmax = std::max(Lmax, L);
      for (int s = 0; s < 2; ++s)
        for (int l = 0; l < L; ++l) CUDA_TRY(ctx->alloc(&p.pyr[s][l], dims[l][0] * dims[l][1]));
      for (int d = 0; d < 2; ++d) {
        TaskState t{};
        t.k = k;
        t.dir = d;
        t.L = L;
        std::memcpy(t.dims, dims, sizeof(dims));
        for (int b = 0; b < 2; ++b) {
          CUDA_TRY(ctx->alloc(&t.UV[b], p.w * p.h));
        }
        for (int b = 0; b < 2; ++b) CUDA_TRY(ctx->alloc(&t.KQ[b], p.w * p.h));
        t.cur = 0;
        t.kc = 0;
        tasks.push_back(t);
      }
    }
    ctx->n_levels_max = Lmax;

    std::vector<HsTask> hs_table;
    std::vector<PrepTask> hp_table;
    std::vector<PyrTask> pyr_table;
    std::vector<int> lists;
    std::vector<Op> plan_scratch;  // the plan is the same for every slot
    std::vector<Op>& plan = sl == 0 ? ctx->plan : plan_scratch;
    plan.push_back({OP_EVENT, 0, 0, 0, 0, 0, 0});
    plan.push_back({OP_EXPAND});
    plan.push_back({OP_CROP});
    plan.push_back({OP_EVENT, 0, 0, 0, 0, 0, 1});
    for (int d = 1; d <= max_depth; ++d) {
      Op op{OP_STATS};
      op.offset = static_cast<int>(lists.size());
      for (int k = 0; k < in->n_pairs; ++k)
        if (depth[k] == d) lists.push_back(k);
      op.count = static_cast<int>(lists.size()) - op.offset;
      plan.push_back(op);
    }
    // the corrected crops + level-0 luma, and with pyr_fuse the first
    // kPyrFused pyramid levels in the same launch
    const int pyr_fused = pyr_fuse_wanted() ? kPyrFused : 1;
    for (int k = 0; k < in->n_pairs; ++k) g.pairs[k].levels = ctx->pair_levels[k];
    {
      Op op{OP_PREP};
      op.fuse = pyr_fused > 1 ? 1 : 0;
      plan.push_back(op);
    }
    plan.push_back({OP_EVENT, 0, 0, 0, 0, 0, 2});

    for (int l = pyr_fused; l < Lmax; ++l) {
      Op op{OP_PYR};
      op.offset = static_cast<int>(pyr_table.size());
      for (int k = 0; k < in->n_pairs; ++k) {
        if (ctx->pair_levels[k] <= l) continue;
        const PairDesc& p = g.pairs[k];
        // recompute dims
        int w = p.w, h = p.h;
        for (int i = 0; i < l - 1; ++i) {
          w = std::max(1, w / 2);
          h = std::max(1, h / 2);
        }
        const int w2 = std::max(1, w / 2), h2 = std::max(1, h / 2);
        for (int s = 0; s < 2; ++s) {
          pyr_table.push_back({p.pyr[s][l - 1], w, h, p.pyr[s][l], w2, h2});
          op.max_px = std::max(op.max_px, w2 * h2);
        }
      }
      op.count = static_cast<int>(pyr_table.size()) - op.offset;
      if (op.count) plan.push_back(op);
    }
    // Each warp iteration (5 per level, flow.cpp:78) is a linearisation (the
    // constants planes) followed by its `sweeps` Jacobi sweeps as nseg
    // launches (segments), ping-ponging two flow buffers per task.  The
    // linearisation is fused into the first segment on the levels where the
    // sweep launcher says it pays (hs_fuse_wanted), else it is a launch of its
    // own; from the second warp iteration on, the previous iteration's last
    // segment linearises it in its epilogue where that is wanted
    // (hs_elin_wanted; the constants then ping-pong between two planes).
    for (int l = Lmax - 1; l >= 0; --l) {
      int n_l = 0, w_l = 0, h_l = 0;
      for (const auto& t : tasks)
        if (l < t.L) {
          ++n_l;
          w_l = std::max(w_l, t.dims[l][0]);
          h_l = std::max(h_l, t.dims[l][1]);
        }
      const std::vector<int> seg_len =
          n_l > 0 ? hs_split(n_l, w_l, h_l, ctx->sweeps) : std::vector<int>(1, ctx->sweeps);
      const int nseg = static_cast<int>(seg_len.size());
      const bool fuse = n_l > 0 && hs_fuse_wanted(n_l, w_l, h_l, seg_len[0]);
      // (a single segment cannot carry both a prologue and an epilogue)
      const bool elin = n_l > 0 && hs_elin_wanted(n_l, w_l, h_l, seg_len[nseg - 1]) &&
                        (nseg >= 2 || !fuse);
      for (int it = 0; it < 5; ++it) {
        const bool lin_done = elin && it > 0;  // by the previous iteration's epilogue
        // u0: zero at the coarsest level's first warp, the coarser flow
        // upsampled at a finer level's first warp, else the previous warp's
        auto lin_mode = [&](const TaskState& t) {
          return (l == t.L - 1 && it == 0) ? 0 : (it == 0 ? 2 : 1);
        };
        if (!fuse && !lin_done) {
          Op pop{OP_HSPREP};
          pop.offset = static_cast<int>(hp_table.size());
          for (auto& t : tasks) {
            if (l >= t.L) continue;
            const PairDesc& p = g.pairs[t.k];
            const int sa = t.dir == 0 ? 0 : 1, sb = 1 - sa;
            PrepTask q{};
            q.a = p.pyr[sa][l];
            q.b = p.pyr[sb][l];
            q.mode = lin_mode(t);
            q.uv_in = t.UV[t.cur];
            q.wc = q.mode == 2 ? t.dims[l + 1][0] : 0;
            q.hc = q.mode == 2 ? t.dims[l + 1][1] : 0;
            q.w = t.dims[l][0];
            q.h = t.dims[l][1];
            q.kq = t.KQ[t.kc];
            if (q.mode != 1) {
              q.uv0_out = t.UV[1 - t.cur];
              t.cur ^= 1;
            }
            hp_table.push_back(q);
            pop.max_w = std::max(pop.max_w, q.w);
            pop.max_h = std::max(pop.max_h, q.h);
          }
          pop.count = static_cast<int>(hp_table.size()) - pop.offset;
          if (pop.count) plan.push_back(pop);
        }
        for (int j = 0; j < nseg; ++j) {
          Op op{OP_HS};
          op.sweeps = seg_len[j];
          op.fuse = (fuse && j == 0 && !lin_done) ? 1
                    : (elin && j == nseg - 1 && it < 4) ? 2
                                                         : 0;
          op.offset = static_cast<int>(hs_table.size());
          for (auto& t : tasks) {
            if (l >= t.L) continue;
            const PairDesc& p = g.pairs[t.k];
            const int sa = t.dir == 0 ? 0 : 1, sb = 1 - sa;
            HsTask h{};
            h.kq = t.KQ[t.kc];
            h.uv_in = t.UV[t.cur];
            h.uv_out = t.UV[1 - t.cur];
            h.w = t.dims[l][0];
            h.h = t.dims[l][1];
            if (op.fuse == 2) {
              h.lin_a = p.pyr[sa][l];
              h.lin_b = p.pyr[sb][l];
              h.kq_next = t.KQ[1 - t.kc];
              t.kc ^= 1;
            } else if (op.fuse == 1) {
              h.lin_a = p.pyr[sa][l];
              h.lin_b = p.pyr[sb][l];
              h.lin_mode = lin_mode(t);
              h.wc = h.lin_mode == 2 ? t.dims[l + 1][0] : 0;
              h.hc = h.lin_mode == 2 ? t.dims[l + 1][1] : 0;
            }
            t.cur ^= 1;
            hs_table.push_back(h);
            op.max_w = std::max(op.max_w, h.w);
            op.max_h = std::max(op.max_h, h.h);
          }
          op.count = static_cast<int>(hs_table.size()) - op.offset;
          if (op.count) plan.push_back(op);
        }
      }
    }
    for (auto& t : tasks) {
      PairDesc& p = g.pairs[t.k];
      p.flow_uv[t.dir] = t.UV[t.cur];
    }
    plan.push_back({OP_EVENT, 0, 0, 0, 0, 0, 3});
    plan.push_back({OP_CANVAS});
    plan.push_back({OP_EVENT, 0, 0, 0, 0, 0, 4});
    plan.push_back({OP_TONE});
    plan.push_back({OP_EVENT, 0, 0, 0, 0, 0, 5});

    // TMA tensor maps of the kq planes (TMA-staged plain segments)
    if (hs_tma_wanted() && !hs_table.empty()) {
      struct alignas(64) Map128 {
        unsigned char b[128];
      };
      std::vector<Map128> maps(hs_table.size());
      for (size_t i = 0; i < hs_table.size(); ++i)
        if (!encode_kq_map(&maps[i], hs_table[i].kq, hs_table[i].w, hs_table[i].h))
          return fail(STITCH_B200_Unsupported, "cuTensorMapEncodeTiled failed");
      Map128* dm = nullptr;
      CUDA_TRY(ctx->alloc(&dm, maps.size()));
      CUDA_TRY(cudaMemcpy(dm, maps.data(), maps.size() * sizeof(Map128), cudaMemcpyHostToDevice));
      for (size_t i = 0; i < hs_table.size(); ++i) hs_table[i].kq_map = dm + i;
    }
    // upload tables + geometry + state
    CUDA_TRY(ctx->alloc(&S.d_hs, hs_table.size() + 1));
    CUDA_TRY(ctx->alloc(&S.d_hp, hp_table.size() + 1));
    CUDA_TRY(ctx->alloc(&S.d_pyr, pyr_table.size() + 1));
    if (!hs_table.empty())
      CUDA_TRY(cudaMemcpy(S.d_hs, hs_table.data(), hs_table.size() * sizeof(HsTask),
                          cudaMemcpyHostToDevice));
    if (!hp_table.empty())
      CUDA_TRY(cudaMemcpy(S.d_hp, hp_table.data(), hp_table.size() * sizeof(PrepTask),
                          cudaMemcpyHostToDevice));
    if (!pyr_table.empty())
      CUDA_TRY(cudaMemcpy(S.d_pyr, pyr_table.data(), pyr_table.size() * sizeof(PyrTask),
                          cudaMemcpyHostToDevice));
    if (sl == 0) {
      CUDA_TRY(ctx->alloc(&ctx->d_lists, lists.size() + 1));
      if (!lists.empty())
        CUDA_TRY(cudaMemcpy(ctx->d_lists, lists.data(), lists.size() * sizeof(int),
                            cudaMemcpyHostToDevice));
    }
    {
      CanvasParams& P = S.cparams;
      P.cw = g.canvas_w;
      P.ch = g.canvas_h;
      P.ref = g.reference;
      P.np = g.n_pairs;
      P.weighting = g.weighting;
      P.offx = g.offx;
      P.offy = g.offy;
      P.projection = g.projection;
      P.lift_sin = g.lift_sin;
      P.lift_cos = g.lift_cos;
      P.lift_h = g.lift_h;
      for (int v = 0; v < g.n_views; ++v) {
        for (int i = 0; i < 9; ++i) P.views[v].inv[i] = g.views[v].inv[i];
        P.views[v].rgba = g.rgba[v];
        P.views[v].w = g.views[v].width;
        P.views[v].h = g.views[v].height;
        for (int i = 0; i < 4; ++i) P.views[v].bbox[i] = g.views[v].bbox[i];
        P.views[v].gap[0] = g.views[v].gap[0];
        P.views[v].gap[1] = g.views[v].gap[1];
        static const int warp_f32 = env_int("STITCH_B200_WARP_F32", 0);
        P.views[v].f32 = warp_f32;
      }
      for (int k = 0; k < g.n_pairs; ++k) {
        const PairDesc& p = g.pairs[k];
        CanvasPair& q = P.pairs[k];
        q.view = p.view;
        q.partner = p.partner;
        q.x0 = p.x0;
        q.y0 = p.y0;
        q.w = p.w;
        q.h = p.h;
        q.theta = p.theta_i;
        for (int s2 = 0; s2 < 2; ++s2) {
          q.crop_raw[s2] = p.crop_raw[s2];
          q.crop_cor[s2] = p.crop_cor[s2];
          q.fuv[s2] = p.flow_uv[s2];
        }
      }
    }
    CUDA_TRY(ctx->alloc(&S.dg, 1));
    CUDA_TRY(cudaMemcpy(S.dg, &g, sizeof(Geometry), cudaMemcpyHostToDevice));
    // device address of this slot's FrameTable::masked (no dereference)
    S.cparams.masked = reinterpret_cast<const int*>(
        reinterpret_cast<const char*>(S.dg) + offsetof(Geometry, in) + offsetof(FrameTable, masked));
    CUDA_TRY(ctx->alloc(&S.dst, 1));
    {
      // identity matrices for every view; the temporal state lives in the
      // shared TemporalState
      std::unique_ptr<DevState> hs(new DevState());
      std::memset(hs.get(), 0, sizeof(DevState));
      char* tbase = reinterpret_cast<char*>(ctx->dtemp);
      hs->windows = reinterpret_cast<PairWindow*>(tbase + offsetof(TemporalState, windows));
      hs->balance = reinterpret_cast<BalanceState*>(tbase + offsetof(TemporalState, balance));
      hs->frame_counter = reinterpret_cast<long long*>(tbase + offsetof(TemporalState, frame_counter));
      for (int v = 0; v < kMaxViews; ++v)
        for (int i = 0; i < 9; ++i) hs->mview[v][i] = (i % 4 == 0) ? 1.0 : 0.0;
      for (int c = 0; c < 3; ++c)
        for (int v = 0; v < 256; ++v) hs->lut[c][v] = static_cast<unsigned char>(v);
      CUDA_TRY(cudaMemcpy(S.dst, hs.get(), sizeof(DevState), cudaMemcpyHostToDevice));
    }
  }
  ctx->hg = ctx->slot[0].hg;
  {
    // canvas class map (geometry only): shared by the slots
    const char* e = getenv("STITCH_B200_CANVAS_CLASS");
    if (!e || atoi(e) != 0) {
      std::uint8_t* cls = nullptr;
      CUDA_TRY(ctx->alloc(&cls, static_cast<size_t>(ctx->n_px)));
      launch_canvas_class(ctx->slot[0].cparams, cls, ctx->stream);
      CUDA_TRY(cudaGetLastError());
      CUDA_TRY(cudaStreamSynchronize(ctx->stream));
      for (int sl = 0; sl < ctx->n_slots; ++sl) ctx->slot[sl].cparams.cls = cls;
    }
  }
  CUDA_TRY(prepare_hs(ctx->sweeps));
  for (int j = 1; j <= ctx->sweeps; ++j) CUDA_TRY(prepare_hs(j));
  for (int sl = 0; sl < ctx->n_slots; ++sl) {
    for (auto& e : ctx->ev[sl]) CUDA_TRY(cudaEventCreate(&e));
    CUDA_TRY(cudaEventCreateWithFlags(&ctx->h2d_done[sl], cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&ctx->comp_done[sl], cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&ctx->d2h_done[sl], cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&ctx->color_done[sl], cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&ctx->canvas_done[sl], cudaEventDisableTiming));
    CUDA_TRY(cudaStreamCreateWithFlags(&ctx->slot[sl].cs, cudaStreamNonBlocking));
  }
  CUDA_TRY(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
  CUDA_TRY(cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking));
  for (auto& e : ctx->ring_ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_ptr_ring), sizeof(FrameTable) * 16,
                         cudaHostAllocDefault));
  CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_report),
                         sizeof(DevReport) * ctx->n_slots, cudaHostAllocDefault));

  // ---- the plan's four segments: front | colour | mid (flow) | back ----
  {
    const auto& pl = ctx->plan;
    const int n = static_cast<int>(pl.size());
    int b1 = -1, b2 = -1, b3 = -1;
    for (int i = 0; i < n; ++i) {
      if (b1 < 0 && pl[i].kind == OP_STATS) b1 = i;
      if (b2 < 0 && pl[i].kind == OP_PREP) b2 = i;
      if (b3 < 0 && pl[i].kind == OP_CANVAS) b3 = i > 0 && pl[i - 1].kind == OP_EVENT ? i - 1 : i;
    }
    if (b2 < 0) b2 = b3;
    if (b1 < 0) b1 = b2;
    ctx->seg_begin[0] = 0;
    ctx->seg_begin[1] = b1;
    ctx->seg_begin[2] = b2;
    ctx->seg_begin[3] = b3;
    ctx->seg_begin[4] = n;
  }
  // ---- capture each slot's segments once ----
  // Programmatic dependent launch: the kernel -> kernel edges of the
  // captured segments become programmatic, so the next kernel launches as
  // soon as the previous one's blocks have all exited instead of after its
  // completion is processed; every frame kernel griddepcontrol.waits for its
  // predecessor (completed, writes visible) before touching global memory.
  // Measured at C2: 905.6 -> 911.7 frames/s, e2e 875 -> 892 (scripts/exp33.sh).
  // STITCH_B200_PDL=0: plain edges; =2: launch when the previous kernel's
  // blocks have all begun (910 frames/s, p50 +0.01 ms).
  static const int pdl = env_int("STITCH_B200_PDL", 1);
  auto make_programmatic = [&](cudaGraph_t gr) -> cudaError_t {
    size_t ne = 0;
    cudaError_t e = cudaGraphGetEdges_v2(gr, nullptr, nullptr, nullptr, &ne);
    if (e != cudaSuccess || ne == 0) return e;
    std::vector<cudaGraphNode_t> from(ne), to(ne);
    std::vector<cudaGraphEdgeData> ed(ne);
    e = cudaGraphGetEdges_v2(gr, from.data(), to.data(), ed.data(), &ne);
    if (e != cudaSuccess) return e;
    for (size_t i = 0; i < ne; ++i) {
      cudaGraphNodeType ta, tb;
      if ((e = cudaGraphNodeGetType(from[i], &ta)) != cudaSuccess) return e;
      if ((e = cudaGraphNodeGetType(to[i], &tb)) != cudaSuccess) return e;
      if (ta != cudaGraphNodeTypeKernel || tb != cudaGraphNodeTypeKernel) continue;
      if ((e = cudaGraphRemoveDependencies_v2(gr, &from[i], &to[i], &ed[i], 1)) != cudaSuccess)
        return e;
      cudaGraphEdgeData pe{};
      pe.type = cudaGraphDependencyTypeProgrammatic;
      pe.from_port = pdl == 2 ? cudaGraphKernelNodePortLaunchCompletion
                              : cudaGraphKernelNodePortProgrammatic;
      if ((e = cudaGraphAddDependencies_v2(gr, &from[i], &to[i], &pe, 1)) != cudaSuccess) return e;
    }
    return cudaSuccess;
  };
  int launches = 0;
  for (int sl = 0; sl < ctx->n_slots; ++sl) {
    SlotRes& S = ctx->slot[sl];
    cudaStream_t s = S.cs;
    launches = 0;
    for (int seg = 0; seg < SlotRes::kSegs; ++seg) {
      if (ctx->seg_begin[seg] == ctx->seg_begin[seg + 1]) continue;
      CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      for (int i = ctx->seg_begin[seg]; i < ctx->seg_begin[seg + 1]; ++i) {
        const Op& op = ctx->plan[i];
        if (op.kind == OP_EVENT)
          cudaEventRecordWithFlags(ctx->ev[sl][op.event], s, cudaEventRecordExternal);
        else
          launches += enqueue_op(ctx.get(), op, s, sl);
      }
      cudaError_t cap_err = cudaStreamEndCapture(s, &S.graph[seg]);
      if (cap_err != cudaSuccess)
        return fail(STITCH_B200_CudaError,
                    std::string("graph capture: ") + cudaGetErrorString(cap_err));
      CUDA_TRY(cudaGetLastError());
      if (pdl) CUDA_TRY(make_programmatic(S.graph[seg]));
      CUDA_TRY(cudaGraphInstantiate(&S.exec[seg], S.graph[seg], 0));
    }
  }
  ctx->launches = launches;
  // the zero fills of ctx->alloc run on the legacy stream, which the context's
  // non-blocking streams do not wait for: settle them before the first frame
  CUDA_TRY(cudaDeviceSynchronize());
  out = std::move(ctx);
  return STITCH_B200_OK;
}

// Point the slot's frame table at this frame's device inputs (pinned ring
// of pointer tables, copied on the slot's stream).
// The slot's per-frame table (inputs, masks, masked flag) from a pinned ring
// entry, stream-ordered before the frame's kernels.  masks: nullptr or per
// view nullptr (unmasked) / device W*H bytes.
int set_frame_pointers(Ctx* ctx, int slot, const std::uint8_t* const* ptrs,
                       const std::uint8_t* const* masks = nullptr) {
  const int r = ctx->ring_pos;
  ctx->ring_pos = (ctx->ring_pos + 1) % 16;
  CUDA_TRY(cudaEventSynchronize(ctx->ring_ev[r]));
  FrameTable* h = ctx->h_ptr_ring + r;
  std::memset(h, 0, sizeof(FrameTable));
  for (int v = 0; v < ctx->hg.n_views; ++v) {
    h->frames[v] = ptrs[v];
    h->masks[v] = masks ? masks[v] : nullptr;
    h->masked |= h->masks[v] != nullptr;
  }
  cudaStream_t cs = ctx->slot[slot].cs;
  CUDA_TRY(cudaMemcpyAsync(&ctx->slot[slot].dg->in, h, sizeof(FrameTable), cudaMemcpyHostToDevice,
                           cs));
  CUDA_TRY(cudaEventRecord(ctx->ring_ev[r], cs));
  return STITCH_B200_OK;
}

void fill_report(Ctx* ctx, int slot, stitch_b200_report* r) {
  const DevReport& d = ctx->h_report[slot];
  std::memset(r, 0, sizeof(*r));
  r->frame_index = d.frame_index;
  r->n_pairs = ctx->hg.n_pairs;
  for (int k = 0; k < ctx->hg.n_pairs; ++k) {
    for (int i = 0; i < 9; ++i) r->color_matrices[k][i] = d.m[k][i];
    r->rank_deficient[k] = d.rank_deficient[k];
  }
  for (int c = 0; c < 3; ++c) {
    r->threshold_m1[c] = d.m1[c];
    r->threshold_m2[c] = d.m2[c];
  }
  r->balanced = d.balanced;
  float t01 = 0, t12 = 0, t23 = 0, t34 = 0, t45 = 0;
  cudaEvent_t* ev = ctx->ev[slot];
  cudaEventElapsedTime(&t01, ev[0], ev[1]);
  cudaEventElapsedTime(&t12, ev[1], ev[2]);
  cudaEventElapsedTime(&t23, ev[2], ev[3]);
  cudaEventElapsedTime(&t34, ev[3], ev[4]);
  cudaEventElapsedTime(&t45, ev[4], ev[5]);
  r->stage_ms[0] = t01;
  r->stage_ms[1] = t12 + t45;
  r->stage_ms[2] = t23;
  r->stage_ms[3] = t34;
}

// Retire the frame occupying `slot` (if any): wait for its download and keep
// its report for a later stitch_b200_wait().
int retire_slot(Ctx* ctx, int slot) {
  if (!ctx->slot_pending[slot]) return STITCH_B200_OK;
  // pageable outputs: ring -> caller.  A download still in flight (a caller
  // waiting right after its submit) is copied chunk by chunk as it lands; a
  // finished one (frames kept in flight) in one batch.
  std::vector<Ctx::OutChunk>& oc = ctx->out_chunks[slot];
  if (!oc.empty()) {
    if (cudaEventQuery(ctx->d2h_done[slot]) == cudaSuccess) {
      std::vector<CopyPool::Job> jobs;
      for (const auto& c : oc) jobs.push_back({c.dst, c.src, c.n});
      ctx->copier->run(jobs);
    } else {
      for (size_t c = 0; c < oc.size(); ++c) {
        CUDA_TRY(cudaEventSynchronize(ctx->out_ev[slot][c]));
        ctx->copier->run({{oc[c].dst, oc[c].src, oc[c].n}});
      }
    }
    oc.clear();
  }
  CUDA_TRY(cudaEventSynchronize(ctx->d2h_done[slot]));
  ctx->user_rgb[slot] = ctx->user_mask[slot] = nullptr;
  stitch_b200_report r;
  fill_report(ctx, slot, &r);
  ctx->done_reports.emplace_back(ctx->slot_ticket[slot], r);
  if (ctx->done_reports.size() > 8) ctx->done_reports.erase(ctx->done_reports.begin());
  ctx->slot_pending[slot] = false;
  return STITCH_B200_OK;
}

// Compute part of one frame on `slot`'s stream: wait until the slot's
// previous download has drained, point the frame table at `dev_in`, then the
// four segment graphs, with the frame-order points of the temporal state
// between slots: the colour solves (3D-M windows) wait for the previous
// frame's, the canvas (threshold history, frame counter) for the previous
// frame's canvas.  Everything else of consecutive frames overlaps.
int enqueue_frame(Ctx* ctx, int slot, const std::uint8_t* const* dev_in,
                  const std::uint8_t* const* dev_masks = nullptr) {
  SlotRes& S = ctx->slot[slot];
  const int prev = (slot + ctx->n_slots - 1) % ctx->n_slots;
  CUDA_TRY(cudaStreamWaitEvent(S.cs, ctx->d2h_done[slot], 0));
  int rc = set_frame_pointers(ctx, slot, dev_in, dev_masks);
  if (rc) return rc;
  if (S.exec[0]) CUDA_TRY(cudaGraphLaunch(S.exec[0], S.cs));
  CUDA_TRY(cudaStreamWaitEvent(S.cs, ctx->color_done[prev], 0));
  if (S.exec[1]) CUDA_TRY(cudaGraphLaunch(S.exec[1], S.cs));
  CUDA_TRY(cudaEventRecord(ctx->color_done[slot], S.cs));
  if (S.exec[2]) CUDA_TRY(cudaGraphLaunch(S.exec[2], S.cs));
  CUDA_TRY(cudaStreamWaitEvent(S.cs, ctx->canvas_done[prev], 0));
  if (S.exec[3]) CUDA_TRY(cudaGraphLaunch(S.exec[3], S.cs));
  CUDA_TRY(cudaEventRecord(ctx->canvas_done[slot], S.cs));
  CUDA_TRY(cudaMemcpyAsync(&ctx->h_report[slot], &S.dst->report, sizeof(DevReport),
                           cudaMemcpyDeviceToHost, S.cs));
  CUDA_TRY(cudaEventRecord(ctx->comp_done[slot], S.cs));
  ctx->last_slot = slot;
  ctx->slot_joined[slot] = false;
  return STITCH_B200_OK;
}

// Wait for all work of the context (uploads, frames, downloads, API stream).
int sync_all(Ctx* ctx) {
  CUDA_TRY(cudaStreamSynchronize(ctx->h2d));
  for (int sl = 0; sl < ctx->n_slots; ++sl) CUDA_TRY(cudaStreamSynchronize(ctx->slot[sl].cs));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->d2h));
  return STITCH_B200_OK;
}

// The slot streams wait for the work enqueued so far on the API stream.
int fork_api_stream(Ctx* ctx) {
  CUDA_TRY(cudaEventRecord(ctx->fork_ev, ctx->stream));
  for (int sl = 0; sl < ctx->n_slots; ++sl)
    CUDA_TRY(cudaStreamWaitEvent(ctx->slot[sl].cs, ctx->fork_ev, 0));
  return STITCH_B200_OK;
}

// The API stream waits for every frame enqueued so far.
int join_api_stream(Ctx* ctx) {
  for (int sl = 0; sl < ctx->n_slots; ++sl)
    if (!ctx->slot_joined[sl]) {
      CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->comp_done[sl], 0));
      ctx->slot_joined[sl] = true;
    }
  return STITCH_B200_OK;
}

// Pinned staging of one slot for pageable caller buffers (first use only).
int ensure_staging(Ctx* ctx, int slot) {
  if (!ctx->copier) {
    const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
    // measured at C2 on a 16-core host: 8 workers 786 fps, 14 workers 826 fps
    // (pinned 895); the copies are bound by host memory bandwidth
    const int n = env_int("STITCH_B200_COPY_THREADS", static_cast<int>(std::min(14u, hw > 4 ? hw - 2 : 2u)));
    ctx->copier.reset(new CopyPool(std::max(0, n)));
  }
  for (int v = 0; v < ctx->hg.n_views; ++v)
    if (!ctx->h_stage_in[slot][v])
      CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_stage_in[slot][v]),
                             ctx->frame_bytes[v], cudaHostAllocDefault));
  if (!ctx->h_stage_rgb[slot])
    CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_stage_rgb[slot]),
                           static_cast<size_t>(ctx->n_px) * 3, cudaHostAllocDefault));
  if (!ctx->h_stage_mask[slot])
    CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_stage_mask[slot]),
                           static_cast<size_t>(ctx->n_px), cudaHostAllocDefault));
  for (cudaEvent_t& e : ctx->out_ev[slot])
    if (!e) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return STITCH_B200_OK;
}

// EmptyProjection of masked frames: every masked view of this frame must
// give at least one valid warped pixel (inside its geometric footprint, which
// holds all of them).  Runs on the upload stream after the mask uploads and
// waits for it: the error must surface before the frame is enqueued.
int check_mask_coverage(Ctx* ctx, int slot, const std::uint8_t* const* dmask) {
  MaskSet ms{};
  unsigned need = 0;
  long long max_px = 0;
  for (int v = 0; v < ctx->hg.n_views; ++v) {
    if (!dmask[v]) continue;
    const int* b = ctx->hg.views[v].bbox;
    ms.view[ms.n] = v;
    ms.mask[ms.n] = dmask[v];
    for (int i = 0; i < 4; ++i) ms.rect[ms.n][i] = b[i];
    max_px = std::max(max_px, static_cast<long long>(b[2] - b[0]) * (b[3] - b[1]));
    need |= 1u << v;
    ++ms.n;
  }
  if (!ms.n) return STITCH_B200_OK;
  if (!ctx->d_cover) {
    void* q = nullptr;
    CUDA_TRY(cudaMalloc(&q, 16));
    ctx->allocs.push_back(q);
    ctx->d_cover = static_cast<unsigned*>(q);
  }
  if (!ctx->h_cover)
    CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_cover), sizeof(unsigned),
                           cudaHostAllocDefault));
  CUDA_TRY(cudaMemsetAsync(ctx->d_cover, 0, sizeof(unsigned), ctx->h2d));
  launch_mask_coverage(ctx->slot[slot].dg, ctx->hg.projection, ms, max_px, ctx->d_cover, ctx->h2d);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(ctx->h_cover, ctx->d_cover, sizeof(unsigned), cudaMemcpyDeviceToHost,
                           ctx->h2d));
  CUDA_TRY(cudaStreamSynchronize(ctx->h2d));
  if ((*ctx->h_cover & need) != need)
    return fail(STITCH_B200_EmptyProjection, "a masked frame projects to no canvas pixel");
  return STITCH_B200_OK;
}

// Host-buffer frame: H2D on the upload stream, compute, D2H on the download
// stream; returns the frame's ticket.  Pinned caller buffers are copied
// directly; pageable ones through the slot's pinned staging ring.
int submit_host(Ctx* ctx, const std::uint8_t* const* frames, std::uint8_t* pano_rgb,
                std::uint8_t* pano_mask, long long* ticket,
                const std::uint8_t* const* masks = nullptr) {
  const int slot = static_cast<int>(ctx->seq % ctx->n_slots);
  int rc = retire_slot(ctx, slot);
  if (rc) return rc;
  for (int v = 0; v < ctx->hg.n_views; ++v)
    if (!frames[v]) return fail(STITCH_B200_InputMismatch, "null frame");
  // pageable inputs / outputs go through the slot's pinned staging ring
  bool idle = true;  // no frame in flight: the synchronous pattern (submit, then wait)
  for (int sl = 0; sl < ctx->n_slots; ++sl) idle = idle && !ctx->slot_pending[sl];
  // (handing pageable buffers to the driver's own staged copies instead was
  // measured slower for the synchronous pattern: 201 vs 257 frames/s at C2)
  bool stage_in[kMaxViews];
  bool any_stage = false;
  for (int v = 0; v < ctx->hg.n_views; ++v) any_stage |= (stage_in[v] = !is_pinned(frames[v]));
  const bool stage_rgb = pano_rgb && !is_pinned(pano_rgb);
  const bool stage_mask = pano_mask && !is_pinned(pano_mask);
  if (any_stage || stage_rgb || stage_mask) {
    rc = ensure_staging(ctx, slot);
    if (rc) return rc;
  }
  // the slot's inputs were last read by its previous frame (retired above,
  // so its staging buffers are free as well)
  CUDA_TRY(cudaStreamWaitEvent(ctx->h2d, ctx->comp_done[slot], 0));
  // An idle pipeline (the synchronous pattern) stages in 4 MiB pieces, each
  // piece's DMA queued as soon as it is copied so it runs while the next one
  // is copied; with frames in flight the copy engine is busy anyway and one
  // batch costs the least.  Measured at C2, synchronous call, pageable input
  // (scripts/sync_stage_modes.py, median ms per call, 14 / 6 / 2 copy
  // workers): 4 MiB pieces 3.05 / 3.01 / 3.19, whole views (the former
  // scheme, STITCH_B200_STAGE_MODE=0) 4.88 / 3.65 / 3.25, one batch (=1)
  // 4.61 / 3.83 / 3.53; pinned input 2.43.
  static const int stage_mode = env_int("STITCH_B200_STAGE_MODE", 2);
  static const size_t stage_chunk =
      static_cast<size_t>(std::max(1, env_int("STITCH_B200_STAGE_CHUNK_MB", 4))) << 20;
  if (any_stage && (!idle || stage_mode == 1)) {
    std::vector<CopyPool::Job> jobs;
    for (int v = 0; v < ctx->hg.n_views; ++v)
      if (stage_in[v]) jobs.push_back({ctx->h_stage_in[slot][v], frames[v], ctx->frame_bytes[v]});
    ctx->copier->run(jobs);
  }
  for (int v = 0; v < ctx->hg.n_views; ++v) {
    if (stage_in[v] && idle && stage_mode == 2) {
      for (size_t o = 0; o < ctx->frame_bytes[v]; o += stage_chunk) {
        const size_t n = std::min(stage_chunk, ctx->frame_bytes[v] - o);
        ctx->copier->run({{ctx->h_stage_in[slot][v] + o, frames[v] + o, n}});
        CUDA_TRY(cudaMemcpyAsync(ctx->d_in[slot][v] + o, ctx->h_stage_in[slot][v] + o, n,
                                 cudaMemcpyHostToDevice, ctx->h2d));
      }
      continue;
    }
    if (stage_in[v] && idle && stage_mode == 0)
      ctx->copier->run({{ctx->h_stage_in[slot][v], frames[v], ctx->frame_bytes[v]}});
    CUDA_TRY(cudaMemcpyAsync(ctx->d_in[slot][v], stage_in[v] ? ctx->h_stage_in[slot][v] : frames[v],
                             ctx->frame_bytes[v], cudaMemcpyHostToDevice, ctx->h2d));
  }
  CUDA_TRY(cudaEventRecord(ctx->h2d_done[slot], ctx->h2d));
  CUDA_TRY(cudaStreamWaitEvent(ctx->slot[slot].cs, ctx->h2d_done[slot], 0));
  // input masks (Frame::mask) travel with the frame to the slot's mask buffers
  const std::uint8_t* dmask[kMaxViews] = {};
  bool any_mask = false;
  for (int v = 0; masks && v < ctx->hg.n_views; ++v) {
    if (!masks[v]) continue;
    any_mask = true;
    const size_t mb = ctx->frame_bytes[v] / 3;
    if (!ctx->d_mask[slot][v]) {
      // no zero fill: a cudaMemset on the legacy stream would not be ordered
      // before the copy below on the (non-blocking) upload stream
      void* q = nullptr;
      CUDA_TRY(cudaMalloc(&q, std::max<size_t>(mb, 16)));
      ctx->allocs.push_back(q);
      ctx->d_mask[slot][v] = static_cast<std::uint8_t*>(q);
    }
    const std::uint8_t* src = masks[v];
    if (!is_pinned(src)) {
      if (!ctx->h_stage_min[slot][v])
        CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_stage_min[slot][v]), mb,
                               cudaHostAllocDefault));
      if (!ctx->copier) {
        rc = ensure_staging(ctx, slot);
        if (rc) return rc;
      }
      ctx->copier->run({{ctx->h_stage_min[slot][v], src, mb}});
      src = ctx->h_stage_min[slot][v];
    }
    CUDA_TRY(cudaMemcpyAsync(ctx->d_mask[slot][v], src, mb, cudaMemcpyHostToDevice, ctx->h2d));
    dmask[v] = ctx->d_mask[slot][v];
  }
  if (any_mask) {
    // warp_frame throws EmptyProjection for a view without one valid warped
    // pixel (geometry.cpp:79), before process_frame touches any state
    // (pipeline.cpp:270-277): the frame fails here, nothing is enqueued
    rc = check_mask_coverage(ctx, slot, dmask);
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(ctx->h2d_done[slot], ctx->h2d));
    CUDA_TRY(cudaStreamWaitEvent(ctx->slot[slot].cs, ctx->h2d_done[slot], 0));
  }
  const std::uint8_t* in[kMaxViews];
  for (int v = 0; v < ctx->hg.n_views; ++v) in[v] = ctx->d_in[slot][v];
  rc = enqueue_frame(ctx, slot, in, any_mask ? dmask : nullptr);
  if (rc) return rc;
  CUDA_TRY(cudaStreamWaitEvent(ctx->d2h, ctx->comp_done[slot], 0));
  const size_t rgb_bytes = static_cast<size_t>(ctx->n_px) * 3, mask_bytes = static_cast<size_t>(ctx->n_px);
  if (pano_rgb && !stage_rgb)
    CUDA_TRY(cudaMemcpyAsync(pano_rgb, ctx->d_out_rgb[slot], rgb_bytes, cudaMemcpyDeviceToHost,
                             ctx->d2h));
  if (pano_mask && !stage_mask)
    CUDA_TRY(cudaMemcpyAsync(pano_mask, ctx->d_out_mask[slot], mask_bytes, cudaMemcpyDeviceToHost,
                             ctx->d2h));
  if (stage_rgb || stage_mask) {
    // chunks of >= 4 MiB, at most kOutChunks in all
    const size_t total = (stage_rgb ? rgb_bytes : 0) + (stage_mask ? mask_bytes : 0);
    const size_t chunk = std::max<size_t>(size_t(4) << 20, (total + Ctx::kOutChunks - 3) / (Ctx::kOutChunks - 2));
    std::vector<Ctx::OutChunk>& oc = ctx->out_chunks[slot];
    oc.clear();
    auto split = [&](std::uint8_t* dst, std::uint8_t* stage, size_t n) {
      for (size_t o = 0; o < n; o += chunk) oc.push_back({dst + o, stage + o, std::min(chunk, n - o)});
    };
    if (stage_rgb) split(pano_rgb, ctx->h_stage_rgb[slot], rgb_bytes);
    const size_t n_rgb_chunks = oc.size();
    if (stage_mask) split(pano_mask, ctx->h_stage_mask[slot], mask_bytes);
    for (size_t c = 0; c < oc.size(); ++c) {
      const bool is_rgb = c < n_rgb_chunks;
      const std::uint8_t* stage0 = is_rgb ? ctx->h_stage_rgb[slot] : ctx->h_stage_mask[slot];
      const std::uint8_t* dev0 = is_rgb ? ctx->d_out_rgb[slot] : ctx->d_out_mask[slot];
      const size_t off = static_cast<size_t>(oc[c].src - stage0);
      CUDA_TRY(cudaMemcpyAsync(const_cast<std::uint8_t*>(oc[c].src), dev0 + off, oc[c].n,
                               cudaMemcpyDeviceToHost, ctx->d2h));
      CUDA_TRY(cudaEventRecord(ctx->out_ev[slot][c], ctx->d2h));
    }
  }
  CUDA_TRY(cudaEventRecord(ctx->d2h_done[slot], ctx->d2h));
  ctx->user_rgb[slot] = stage_rgb ? pano_rgb : nullptr;
  ctx->user_mask[slot] = stage_mask ? pano_mask : nullptr;
  ctx->slot_ticket[slot] = ctx->seq;
  ctx->slot_pending[slot] = true;
  if (ticket) *ticket = ctx->seq;
  ++ctx->seq;
  return STITCH_B200_OK;
}

int wait_ticket(Ctx* ctx, long long ticket, stitch_b200_report* report) {
  for (auto& d : ctx->done_reports)
    if (d.first == ticket) {
      if (report) *report = d.second;
      return STITCH_B200_OK;
    }
  for (int sl = 0; sl < ctx->n_slots; ++sl)
    if (ctx->slot_pending[sl] && ctx->slot_ticket[sl] == ticket) {
      int rc = retire_slot(ctx, sl);
      if (rc) return rc;
      return wait_ticket(ctx, ticket, report);
    }
  return fail(STITCH_B200_MissingState, "unknown or expired ticket");
}

}  // namespace

extern "C" {

const char* stitch_b200_last_error(void) { return g_last_error.c_str(); }

const char* stitch_b200_version(void) { return "stitch_b200 0.1 (sm_100a)"; }

void stitch_b200_config_defaults(stitch_b200_config* c) { hg_ns::config_defaults(c); }

int stitch_b200_create(const stitch_b200_init* init, int device, stitch_b200_ctx** out) {
  *out = nullptr;
  std::unique_ptr<Ctx> ctx;
  int rc = build_context(init, device, nullptr, ctx);
  if (rc) return rc;
  *out = new stitch_b200_ctx{std::move(ctx)};
  return STITCH_B200_OK;
}

// refine_pair (pipeline.cpp:114-179) for every pair, on the first frames
// warped with the unrefined maps: detection, description and matching on
// the device (features_kernels.cu), back-projection, RANSAC, the Jacobian
// transport and refine_homography on the host.  maps / invs of refined views
// are replaced; warn[k] = PairState::refine_warning.
static int refine_maps(int device, const stitch_b200_config* cfg, const uint8_t* const* frames,
                       const uint8_t* const* masks,
                       const Geometry& geom, const std::vector<PairGeometry>& pgeo,
                       const std::vector<hg_ns::PairSpec>& pairs, std::vector<hg_ns::Mat3>& maps,
                       std::vector<hg_ns::Mat3>& invs, std::vector<int>& warn) {
  CUDA_TRY(cudaSetDevice(device));
  const int cw = geom.canvas_w, ch = geom.canvas_h;
  if (ch >= (1 << 13) || cw >= (1 << 15))
    return fail(STITCH_B200_Unsupported, "refinement supports canvases below 32768 x 8192");
  cudaStream_t s = nullptr;
  CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct Guard {
    cudaStream_t s;
    std::vector<void*> p;
    ~Guard() {
      for (void* q : p) cudaFree(q);
      cudaStreamDestroy(s);
    }
  } gd{s, {}};
  auto dalloc = [&](void** q, size_t n) -> cudaError_t {
    cudaError_t e = cudaMalloc(q, n + 16);
    if (e == cudaSuccess) gd.p.push_back(*q);
    return e;
  };
  void* dg = nullptr;
  CUDA_TRY(dalloc(&dg, sizeof(Geometry)));
  CUDA_TRY(cudaMemcpyAsync(dg, &geom, sizeof(Geometry), cudaMemcpyHostToDevice, s));
  const size_t P = static_cast<size_t>(cw) * ch;
  void *wrgb = nullptr, *wmask = nullptr;
  CUDA_TRY(dalloc(&wrgb, 3 * P));
  CUDA_TRY(dalloc(&wmask, P));
  // warp_frame of the first frames (the per-frame sampler's arithmetic) and
  // the integral image of each warped view taking part in a pair
  std::vector<std::unique_ptr<FeatView>> fv(cfg->n_views);
  for (const auto& pr : pairs)
    for (int v : {pr.view, pr.partner}) {
      if (fv[v]) continue;
      const size_t npx = static_cast<size_t>(cfg->width[v]) * cfg->height[v];
      void *src = nullptr, *rgba = nullptr;
      CUDA_TRY(dalloc(&src, 3 * npx));
      CUDA_TRY(dalloc(&rgba, 4 * npx));
      CUDA_TRY(cudaMemcpyAsync(src, frames[v], 3 * npx, cudaMemcpyHostToDevice, s));
      void* dm = nullptr;  // the first frame's mask (Frame::mask) as the RGBA alpha
      if (masks && masks[v]) {
        CUDA_TRY(dalloc(&dm, npx));
        CUDA_TRY(cudaMemcpyAsync(dm, masks[v], npx, cudaMemcpyHostToDevice, s));
      }
      launch_expand_one(static_cast<const std::uint8_t*>(src), static_cast<uchar4*>(rgba),
                        static_cast<long long>(npx), s, static_cast<const std::uint8_t*>(dm));
      launch_warp_view(static_cast<const Geometry*>(dg), v, static_cast<const uchar4*>(rgba),
                       static_cast<std::uint8_t*>(wrgb), static_cast<std::uint8_t*>(wmask), s,
                       dm != nullptr);
      CUDA_TRY(cudaGetLastError());
      fv[v].reset(new FeatView());
      CUDA_TRY(fv[v]->build(static_cast<const std::uint8_t*>(wrgb), cw, ch, s));
    }
  const int canvas_r[4] = {0, 0, cw, ch};
  warn.assign(pairs.size(), 1);
  for (size_t k = 0; k < pairs.size(); ++k) {
    const int view = pairs[k].view, partner = pairs[k].partner;
    int search[4];
    hg_ns::broaden(pgeo[k].bounds, cfg->refine_margin, canvas_r, search);
    if (search[2] - search[0] < 32 || search[3] - search[1] < 32) continue;  // RegionTooSmall
    std::vector<FeatPoint> kv, kr;
    std::vector<float> dv, dr;
    CUDA_TRY(fv[view]->detect_describe(search[0], search[1], search[2], search[3],
                                       cfg->detect_threshold, kv, dv, s));
    CUDA_TRY(fv[partner]->detect_describe(search[0], search[1], search[2], search[3],
                                          cfg->detect_threshold, kr, dr, s));
    if (kv.empty() || kr.empty()) continue;
    std::vector<int> best_b, best_a;
    std::vector<double> best_dist;
    CUDA_TRY(feat_match(dv, dr, static_cast<int>(kv.size()), static_cast<int>(kr.size()),
                        cfg->match_ratio, best_b, best_dist, best_a, s));
    const hg_ns::Mat3 map = maps[view];
    hg_ns::Mat3 inv;
    int rc = hg_ns::homography_inverse(map, inv);  // Homography::inverse
    if (rc) return fail(rc, "singular map during refinement");
    std::vector<hg_ns::MatchPt> m;
    for (size_t a = 0; a < kv.size(); ++a) {
      const int b = best_b[a];
      if (b < 0 || best_a[b] != static_cast<int>(a)) continue;  // cross-check
      hg_ns::MatchPt mp;
      hg_ns::homography_apply(inv, kv[a].x + geom.offx, kv[a].y + geom.offy, mp.ax, mp.ay);
      hg_ns::homography_apply(inv, kr[b].x + geom.offx, kr[b].y + geom.offy, mp.bx, mp.by);
      mp.distance = best_dist[a];
      m.push_back(mp);
    }
    hg_ns::ScaleShift fit;
    rc = hg_ns::ransac_scale_translation(m, cfg->ransac_iters, cfg->inlier_px, 0.5, 2.0,
                                         cfg->seed + static_cast<std::uint64_t>(view), fit);
    if (rc) continue;  // InsufficientMatches / NoConsensus: keep the unrefined map
    // translation carried to the plane with the local Jacobian at the
    // overlap centre (pipeline.cpp:98-112, 160-170)
    const int* bb = pgeo[k].bounds;
    const double cx = geom.offx + bb[0] + (bb[2] - bb[0]) / 2.0;
    const double cy = geom.offy + bb[1] + (bb[3] - bb[1]) / 2.0;
    double ax, ay;
    hg_ns::homography_apply(inv, cx, cy, ax, ay);
    const double eps = 1e-4;
    double xp0, yp0, xm0, ym0, xp1, yp1, xm1, ym1;
    hg_ns::homography_apply(map, ax + eps, ay, xp0, yp0);
    hg_ns::homography_apply(map, ax - eps, ay, xm0, ym0);
    hg_ns::homography_apply(map, ax, ay + eps, xp1, yp1);
    hg_ns::homography_apply(map, ax, ay - eps, xm1, ym1);
    const double j00 = (xp0 - xm0) / (2 * eps), j10 = (yp0 - ym0) / (2 * eps);
    const double j01 = (xp1 - xm1) / (2 * eps), j11 = (yp1 - ym1) / (2 * eps);
    const double tx = j00 * fit.t_x + j01 * fit.t_y;
    const double ty = j10 * fit.t_x + j11 * fit.t_y;
    // refine_homography (geometry.cpp:135-145): T(tx, ty) * H * S(sx, sy)
    const hg_ns::Mat3 t = {1, 0, tx, 0, 1, ty, 0, 0, 1};
    const hg_ns::Mat3 sc = {fit.s_x, 0, 0, 0, fit.s_y, 0, 0, 0, 1};
    hg_ns::Mat3 th, ths, refined;
    hg_ns::mul3(t, map, th);
    hg_ns::mul3(th, sc, ths);
    rc = hg_ns::homography_from_matrix(ths, refined);
    if (rc) return fail(rc, "refinement produced a singular map");
    maps[view] = refined;
    hg_ns::inverse3(refined, invs[view]);  // pipeline.cpp:40
    warn[k] = 0;
  }
  return STITCH_B200_OK;
}

// The first frames expanded to RGBA with their masks as alpha, on the device
// (masked views only), for the pair geometry of masked first frames.
struct FirstFrames {
  std::vector<void*> bufs;
  std::vector<const uchar4*> rgba;
  ~FirstFrames() {
    for (void* p : bufs) cudaFree(p);
  }
};

static int upload_masked_first(int device, const stitch_b200_config* cfg,
                               const uint8_t* const* frames, const uint8_t* const* masks,
                               FirstFrames& ff) {
  CUDA_TRY(cudaSetDevice(device));
  ff.rgba.assign(static_cast<size_t>(cfg->n_views), nullptr);
  for (int v = 0; v < cfg->n_views; ++v) {
    if (!masks[v]) continue;
    const size_t npx = static_cast<size_t>(cfg->width[v]) * cfg->height[v];
    void *src = nullptr, *dm = nullptr, *rgba = nullptr;
    CUDA_TRY(cudaMalloc(&src, 3 * npx + 16));
    ff.bufs.push_back(src);
    CUDA_TRY(cudaMalloc(&dm, npx + 16));
    ff.bufs.push_back(dm);
    CUDA_TRY(cudaMalloc(&rgba, 4 * npx + 16));
    ff.bufs.push_back(rgba);
    CUDA_TRY(cudaMemcpy(src, frames[v], 3 * npx, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(dm, masks[v], npx, cudaMemcpyHostToDevice));
    launch_expand_one(static_cast<const std::uint8_t*>(src), static_cast<uchar4*>(rgba),
                      static_cast<long long>(npx), 0, static_cast<const std::uint8_t*>(dm));
    CUDA_TRY(cudaGetLastError());
    ff.rgba[v] = static_cast<const uchar4*>(rgba);
  }
  CUDA_TRY(cudaDeviceSynchronize());
  return STITCH_B200_OK;
}

static int initialize_impl(const stitch_b200_config* cfg, const uint8_t* const* frames, int device,
                           stitch_b200_ctx** out, const uint8_t* const* masks = nullptr) {
  *out = nullptr;
  if (cfg->refine_enabled && !frames)
    return fail(STITCH_B200_ConfigurationError,
                "feature refinement needs the first frames: use stitch_b200_initialize_frames");
  if (cfg->refine_enabled && cfg->projection == 1)
    return fail(STITCH_B200_Unsupported, "feature refinement serves the planar canvas");
  if (cfg->n_views < 2 || cfg->n_views > kMaxViews)
    return fail(STITCH_B200_ConfigurationError, "n_views must be in [2, 16]");
  if (cfg->reference < 0 || cfg->reference >= cfg->n_views)
    return fail(STITCH_B200_ConfigurationError, "reference view index out of range");
  std::vector<hg_ns::Mat3> maps(cfg->n_views), invs(cfg->n_views);
  hg_ns::Canvas canvas;
  double cyl_f = 0.0;
  if (cfg->projection == 1) {
    // cylindrical 360-degree canvas (extension): A_v = K_v R_v R_ref^T
    cyl_f = cfg->cyl_focal > 0.0 ? cfg->cyl_focal : cfg->cams[cfg->reference].fx;
    hg_ns::cylinder_maps(*cfg, invs);
    canvas = hg_ns::cylinder_canvas(*cfg, cyl_f);
  } else {
    // camera homographies and pairwise maps (pipeline.cpp:219-229)
    std::vector<hg_ns::Mat3> cam(cfg->n_views);
    std::vector<std::pair<int, int>> sizes;
    for (int v = 0; v < cfg->n_views; ++v) {
      int rc = hg_ns::planar_homography(cfg->cams[v], cam[v]);
      if (rc) return fail(rc, "camera homography failed (rotation or degenerate pose)");
    }
    for (int v = 0; v < cfg->n_views; ++v) {
      int rc = hg_ns::pairwise_homography(cam[cfg->reference], cam[v], maps[v]);
      if (rc) return fail(rc, "singular pairwise homography");
      sizes.emplace_back(cfg->width[v], cfg->height[v]);
      hg_ns::inverse3(maps[v], invs[v]);  // pipeline.cpp:40
    }
    canvas = hg_ns::compute_canvas(maps, sizes);  // pipeline.cpp:231
  }
  stitch_b200_init in{};
  in.canvas_width = canvas.width;
  in.canvas_height = canvas.height;
  in.canvas_offset[0] = canvas.offx;
  in.canvas_offset[1] = canvas.offy;
  in.n_views = cfg->n_views;
  in.reference = cfg->reference;
  in.projection = cfg->projection == 1 ? 1 : 0;
  in.cyl_focal = cyl_f;
  for (int v = 0; v < cfg->n_views; ++v) {
    in.view_width[v] = cfg->width[v];
    in.view_height[v] = cfg->height[v];
    for (int i = 0; i < 9; ++i) in.inv_maps[v][i] = invs[v][i];
  }
  in.window_capacity = cfg->window_capacity;
  in.lambda = cfg->lambda;
  in.gamma_dark = cfg->gamma_dark;
  in.gamma_bright = cfg->gamma_bright;
  in.target_black = cfg->target_black;
  in.target_white = cfg->target_white;
  in.flow_levels = cfg->flow_levels;
  in.flow_iterations = cfg->flow_iterations;
  in.smoothness = cfg->smoothness;
  in.fuse_weighting = cfg->fuse_weighting;
  if (canvas.width <= 0 || canvas.height <= 0 ||
      static_cast<long long>(canvas.width) * canvas.height > (1ll << 31))
    return fail(STITCH_B200_ConfigurationError, "canvas size out of range");
  // rebuild_pair_geometry (pipeline.cpp:181-205), all on the device: warp
  // masks, view footprints, overlap bounds, chamfer blend weights.
  Geometry g{};
  fill_views(g, &in);
  const int topo = (cfg->projection == 1 && cfg->topology == 0) ? 3 : cfg->topology;
  const auto pairs = hg_ns::build_pairs(cfg->n_views, cfg->reference, topo);
  if (static_cast<int>(pairs.size()) > kMaxPairs)
    return fail(STITCH_B200_ConfigurationError, "too many pairs");
  std::vector<std::pair<int, int>> vp;
  for (const auto& pr : pairs) vp.emplace_back(pr.view, pr.partner);
  std::vector<ViewFootprint> views;
  std::vector<PairGeometry> pgeo;
  // masked first frames decide the pair geometry (rebuild_pair_geometry warps
  // first_frames, pipeline.cpp:181-205)
  bool any_mask = false;
  for (int v = 0; frames && masks && v < cfg->n_views; ++v) any_mask |= masks[v] != nullptr;
  FirstFrames ff;
  if (any_mask) {
    int rc0 = upload_masked_first(device, cfg, frames, masks, ff);
    if (rc0) return rc0;
  }
  const std::vector<const uchar4*>* first_rgba = any_mask ? &ff.rgba : nullptr;
  // rebuild_pair_geometry warps every first frame before it looks at any
  // overlap: a masked first frame without one valid warped pixel is
  // EmptyProjection (geometry.cpp:79), before NoOverlap
  auto masked_empty = [&]() {
    for (const ViewFootprint& f : views)
      if (f.masked_empty)
        return fail(STITCH_B200_EmptyProjection, "a masked first frame projects to no canvas pixel");
    return static_cast<int>(STITCH_B200_OK);
  };
  int rc = init_geometry(device, g, make_lift(&in), cfg->n_views, vp, views, pgeo, first_rgba);
  if (rc) return rc;
  rc = masked_empty();
  if (rc) return rc;
  std::vector<int> warn(pairs.size(), 0);
  if (cfg->refine_enabled) {
    for (size_t k = 0; k < pairs.size(); ++k)
      if (!pgeo[k].ok) return fail(STITCH_B200_ConfigurationError, "adjacent views do not overlap");
    rc = refine_maps(device, cfg, frames, any_mask ? masks : nullptr, g, pgeo, pairs, maps, invs,
                     warn);
    if (rc) return rc;
    // refinement moved the maps: bounds and weights shift (pipeline.cpp:254);
    // the canvas is kept (the reference computes it before refining)
    for (int v = 0; v < cfg->n_views; ++v)
      for (int i = 0; i < 9; ++i) in.inv_maps[v][i] = invs[v][i];
    fill_views(g, &in);
    rc = init_geometry(device, g, make_lift(&in), cfg->n_views, vp, views, pgeo, first_rgba);
    if (rc) return rc;
    rc = masked_empty();
    if (rc) return rc;
  }
  in.n_pairs = static_cast<int>(pairs.size());
  for (size_t k = 0; k < pairs.size(); ++k) {
    if (!pgeo[k].ok) return fail(STITCH_B200_ConfigurationError, "adjacent views do not overlap");
    stitch_b200_pair& p = in.pairs[k];
    p.view = pairs[k].view;
    p.partner = pairs[k].partner;
    p.x0 = pgeo[k].bounds[0];
    p.y0 = pgeo[k].bounds[1];
    p.x1 = pgeo[k].bounds[2];
    p.y1 = pgeo[k].bounds[3];
    p.theta_i = pgeo[k].theta.data();
  }
  std::unique_ptr<Ctx> ctx;
  rc = build_context(&in, device, &views, ctx);
  if (rc) return rc;
  ctx->refine_warning = warn;
  *out = new stitch_b200_ctx{std::move(ctx)};
  return STITCH_B200_OK;
}

int stitch_b200_initialize(const stitch_b200_config* cfg, int device, stitch_b200_ctx** out) {
  return initialize_impl(cfg, nullptr, device, out);
}

int stitch_b200_initialize_frames(const stitch_b200_config* cfg, const uint8_t* const* frames,
                                  int device, stitch_b200_ctx** out) {
  if (!frames) return fail(STITCH_B200_ConfigurationError, "frames must not be NULL");
  return initialize_impl(cfg, frames, device, out);
}

int stitch_b200_initialize_frames_masked(const stitch_b200_config* cfg,
                                         const uint8_t* const* frames, const uint8_t* const* masks,
                                         int device, stitch_b200_ctx** out) {
  if (!frames) return fail(STITCH_B200_ConfigurationError, "frames must not be NULL");
  return initialize_impl(cfg, frames, device, out, masks);
}

static int carry_into(stitch_b200_ctx* h, std::unique_ptr<Ctx>& fresh);

int stitch_b200_rerefine_masked(stitch_b200_ctx* h, const stitch_b200_config* cfg,
                                const uint8_t* const* frames, const uint8_t* const* masks) {
  if (!frames) return fail(STITCH_B200_ConfigurationError, "frames must not be NULL");
  stitch_b200_ctx* fresh = nullptr;
  int rc = initialize_impl(cfg, frames, h->c->device, &fresh, masks);
  if (rc) return rc;
  std::unique_ptr<stitch_b200_ctx> guard(fresh);
  if (fresh->c->hg.n_pairs != h->c->hg.n_pairs)
    return fail(STITCH_B200_ConfigurationError, "re-refinement must keep the pair set");
  std::unique_ptr<Ctx> f = std::move(fresh->c);
  return carry_into(h, f);
}

int stitch_b200_rerefine(stitch_b200_ctx* h, const stitch_b200_config* cfg,
                         const uint8_t* const* frames) {
  return stitch_b200_rerefine_masked(h, cfg, frames, nullptr);
}

int stitch_b200_refine_warning(const stitch_b200_ctx* h, int k) {
  const Ctx* ctx = h->c.get();
  if (k < 0 || k >= ctx->hg.n_pairs) return 0;
  return k < static_cast<int>(ctx->refine_warning.size()) ? ctx->refine_warning[k] : 0;
}

// Replace a context by a freshly built one, carrying the 3D-M windows,
// threshold history and frame counter over (pipeline.cpp:399-405).
static int carry_into(stitch_b200_ctx* h, std::unique_ptr<Ctx>& fresh) {
  Ctx* ctx = h->c.get();
  int rc = sync_all(ctx);
  if (rc) return rc;
  // retire every pending host-path frame so its report survives the swap,
  // and keep ticket numbers monotonic: tickets issued before the swap stay
  // waitable and can never alias a later frame
  for (int sl = 0; sl < ctx->n_slots; ++sl) {
    rc = retire_slot(ctx, sl);
    if (rc) return rc;
  }
  fresh->done_reports = std::move(ctx->done_reports);
  fresh->seq = ctx->seq;
  // carry windows, threshold history and the frame counter over
  // (pipeline.cpp:399-405)
  CUDA_TRY(cudaMemcpy(fresh->dtemp, ctx->dtemp, sizeof(TemporalState), cudaMemcpyDeviceToDevice));
  h->c = std::move(fresh);  // the old context is released here
  return STITCH_B200_OK;
}

int stitch_b200_update_geometry(stitch_b200_ctx* h, const stitch_b200_init* init) {
  Ctx* ctx = h->c.get();
  if (init->n_pairs != ctx->hg.n_pairs)
    return fail(STITCH_B200_ConfigurationError, "re-refinement must keep the pair set");
  std::unique_ptr<Ctx> fresh;
  int rc = build_context(init, ctx->device, nullptr, fresh);
  if (rc) return rc;
  return carry_into(h, fresh);
}

int stitch_b200_camera_maps(const stitch_b200_config* cfg, double* maps) {
  if (cfg->n_views < 2 || cfg->n_views > kMaxViews)
    return fail(STITCH_B200_ConfigurationError, "n_views must be in [2, 16]");
  if (cfg->reference < 0 || cfg->reference >= cfg->n_views)
    return fail(STITCH_B200_ConfigurationError, "reference view index out of range");
  std::vector<hg_ns::Mat3> cam(cfg->n_views);
  for (int v = 0; v < cfg->n_views; ++v) {
    int rc = hg_ns::planar_homography(cfg->cams[v], cam[v]);
    if (rc) return fail(rc, "camera homography failed (rotation or degenerate pose)");
  }
  for (int v = 0; v < cfg->n_views; ++v) {
    hg_ns::Mat3 m;
    int rc = hg_ns::pairwise_homography(cam[cfg->reference], cam[v], m);
    if (rc) return fail(rc, "singular pairwise homography");
    for (int i = 0; i < 9; ++i) maps[9 * v + i] = m[i];
  }
  return STITCH_B200_OK;
}

int stitch_b200_update_maps(stitch_b200_ctx* h, const double* maps) {
  Ctx* ctx = h->c.get();
  if (ctx->init.projection != 0)
    return fail(STITCH_B200_Unsupported, "update_maps serves the planar canvas");
  stitch_b200_init in = ctx->init;
  const int n = in.n_views;
  std::vector<hg_ns::Mat3> fw(n), inv(n);
  std::vector<std::pair<int, int>> sizes;
  for (int v = 0; v < n; ++v) {
    for (int i = 0; i < 9; ++i) fw[v][i] = maps[9 * v + i];
    hg_ns::inverse3(fw[v], inv[v]);  // pipeline.cpp:40
    sizes.emplace_back(in.view_width[v], in.view_height[v]);
  }
  const hg_ns::Canvas canvas = hg_ns::compute_canvas(fw, sizes);  // pipeline.cpp:231
  if (canvas.width <= 0 || canvas.height <= 0 ||
      static_cast<long long>(canvas.width) * canvas.height > (1ll << 31))
    return fail(STITCH_B200_ConfigurationError, "canvas size out of range");
  in.canvas_width = canvas.width;
  in.canvas_height = canvas.height;
  in.canvas_offset[0] = canvas.offx;
  in.canvas_offset[1] = canvas.offy;
  for (int v = 0; v < n; ++v)
    for (int i = 0; i < 9; ++i) in.inv_maps[v][i] = inv[v][i];
  Geometry g{};
  fill_views(g, &in);
  std::vector<std::pair<int, int>> vp;
  for (int k = 0; k < in.n_pairs; ++k) vp.emplace_back(in.pairs[k].view, in.pairs[k].partner);
  std::vector<ViewFootprint> views;
  std::vector<PairGeometry> pgeo;
  int rc = init_geometry(ctx->device, g, make_lift(&in), n, vp, views, pgeo);
  if (rc) return rc;
  for (int k = 0; k < in.n_pairs; ++k) {
    if (!pgeo[k].ok) return fail(STITCH_B200_ConfigurationError, "adjacent views do not overlap");
    stitch_b200_pair& p = in.pairs[k];
    p.x0 = pgeo[k].bounds[0];
    p.y0 = pgeo[k].bounds[1];
    p.x1 = pgeo[k].bounds[2];
    p.y1 = pgeo[k].bounds[3];
    p.theta_i = pgeo[k].theta.data();
  }
  std::unique_ptr<Ctx> fresh;
  rc = build_context(&in, ctx->device, &views, fresh);
  if (rc) return rc;
  return carry_into(h, fresh);
}

void stitch_b200_destroy(stitch_b200_ctx* h) { delete h; }

int stitch_b200_canvas(const stitch_b200_ctx* hd, int* w, int* h, double* ox, double* oy) {
  const Ctx* ctx = hd->c.get();
  if (w) *w = ctx->hg.canvas_w;
  if (h) *h = ctx->hg.canvas_h;
  if (ox) *ox = ctx->hg.offx;
  if (oy) *oy = ctx->hg.offy;
  return STITCH_B200_OK;
}

int stitch_b200_n_pairs(const stitch_b200_ctx* h) { return h->c->hg.n_pairs; }

int stitch_b200_n_views(const stitch_b200_ctx* h) { return h->c->hg.n_views; }

int stitch_b200_slots(const stitch_b200_ctx* h) { return h->c->n_slots; }

int stitch_b200_view_size(const stitch_b200_ctx* h, int view, int* width, int* height) {
  const Ctx* ctx = h->c.get();
  if (view < 0 || view >= ctx->hg.n_views)
    return fail(STITCH_B200_InputMismatch, "view index out of range");
  if (width) *width = ctx->hg.views[view].width;
  if (height) *height = ctx->hg.views[view].height;
  return STITCH_B200_OK;
}

int stitch_b200_check_frames(const stitch_b200_ctx* h, int n, const int* widths,
                             const int* heights, const uint8_t* const* masks) {
  const Ctx* ctx = h->c.get();
  if (n != ctx->hg.n_views)
    return fail(STITCH_B200_ConfigurationError, "frame count does not match configured views");
  for (int v = 0; v < n; ++v) {
    const int w = ctx->hg.views[v].width, ht = ctx->hg.views[v].height;
    if (widths[v] != w || heights[v] != ht) {
      char msg[160];
      std::snprintf(msg, sizeof(msg), "frame %d is %dx%d, the context was initialized for %dx%d",
                    v, widths[v], heights[v], w, ht);
      return fail(STITCH_B200_InputMismatch, msg);
    }
  }
  (void)masks;  // masked frames are supported (stitch_b200_process_masked / submit_masked)
  return STITCH_B200_OK;
}

int stitch_b200_set_error(int code, const char* what) { return fail(code, what ? what : ""); }

int stitch_b200_get_pair(const stitch_b200_ctx* h, int k, stitch_b200_pair* pair,
                         float* theta_out) {
  const Ctx* ctx = h->c.get();
  if (k < 0 || k >= ctx->hg.n_pairs) return fail(STITCH_B200_ConfigurationError, "bad pair index");
  *pair = ctx->init.pairs[k];
  if (theta_out)
    std::memcpy(theta_out, ctx->theta_host[k].data(), ctx->theta_host[k].size() * sizeof(float));
  return STITCH_B200_OK;
}

int stitch_b200_view_bbox(const stitch_b200_ctx* h, int view, int bbox[4]) {
  const Ctx* ctx = h->c.get();
  if (view < 0 || view >= ctx->hg.n_views) return fail(STITCH_B200_ConfigurationError, "bad view");
  for (int i = 0; i < 4; ++i) bbox[i] = ctx->hg.views[view].bbox[i];
  return STITCH_B200_OK;
}

int stitch_b200_get_inv_map(const stitch_b200_ctx* h, int view, double inv[9]) {
  const Ctx* ctx = h->c.get();
  if (view < 0 || view >= ctx->hg.n_views) return fail(STITCH_B200_ConfigurationError, "bad view");
  for (int i = 0; i < 9; ++i) inv[i] = ctx->hg.views[view].inv[i];
  return STITCH_B200_OK;
}

int stitch_b200_process(stitch_b200_ctx* h, const uint8_t* const* frames, uint8_t* pano_rgb,
                        uint8_t* pano_mask, stitch_b200_report* report) {
  Ctx* ctx = h->c.get();
  CUDA_TRY(cudaSetDevice(ctx->device));
  long long ticket = -1;
  int rc = submit_host(ctx, frames, pano_rgb, pano_mask, &ticket);
  if (rc) return rc;
  stitch_b200_report tmp;
  return wait_ticket(ctx, ticket, report ? report : &tmp);
}

int stitch_b200_submit(stitch_b200_ctx* h, const uint8_t* const* frames, uint8_t* pano_rgb,
                       uint8_t* pano_mask, long long* ticket) {
  Ctx* ctx = h->c.get();
  CUDA_TRY(cudaSetDevice(ctx->device));
  return submit_host(ctx, frames, pano_rgb, pano_mask, ticket);
}

int stitch_b200_process_masked(stitch_b200_ctx* h, const uint8_t* const* frames,
                               const uint8_t* const* masks, uint8_t* pano_rgb, uint8_t* pano_mask,
                               stitch_b200_report* report) {
  Ctx* ctx = h->c.get();
  CUDA_TRY(cudaSetDevice(ctx->device));
  long long ticket = -1;
  int rc = submit_host(ctx, frames, pano_rgb, pano_mask, &ticket, masks);
  if (rc) return rc;
  stitch_b200_report tmp;
  return wait_ticket(ctx, ticket, report ? report : &tmp);
}

int stitch_b200_submit_masked(stitch_b200_ctx* h, const uint8_t* const* frames,
                              const uint8_t* const* masks, uint8_t* pano_rgb, uint8_t* pano_mask,
                              long long* ticket) {
  Ctx* ctx = h->c.get();
  CUDA_TRY(cudaSetDevice(ctx->device));
  return submit_host(ctx, frames, pano_rgb, pano_mask, ticket, masks);
}

int stitch_b200_wait(stitch_b200_ctx* h, long long ticket, stitch_b200_report* report) {
  Ctx* ctx = h->c.get();
  CUDA_TRY(cudaSetDevice(ctx->device));
  stitch_b200_report tmp;
  return wait_ticket(ctx, ticket, report ? report : &tmp);
}

int stitch_b200_process_device(stitch_b200_ctx* h, const uint8_t* const* dev_frames,
                               stitch_b200_report* report) {
  Ctx* ctx = h->c.get();
  CUDA_TRY(cudaSetDevice(ctx->device));
  const int slot = static_cast<int>(ctx->seq % ctx->n_slots);
  int rc = retire_slot(ctx, slot);
  if (rc) return rc;
  // stream-ordered on the API stream: inputs written there are seen, and
  // work enqueued there afterwards sees the outputs
  rc = fork_api_stream(ctx);
  if (rc) return rc;
  rc = enqueue_frame(ctx, slot, dev_frames);
  if (rc) return rc;
  rc = join_api_stream(ctx);
  if (rc) return rc;
  ++ctx->seq;
  if (report) {
    CUDA_TRY(cudaEventSynchronize(ctx->comp_done[slot]));
    fill_report(ctx, slot, report);
  }
  return STITCH_B200_OK;
}

int stitch_b200_process_device_async(stitch_b200_ctx* h, const uint8_t* const* dev_frames) {
  Ctx* ctx = h->c.get();
  CUDA_TRY(cudaSetDevice(ctx->device));
  const int slot = static_cast<int>(ctx->seq % ctx->n_slots);
  int rc = retire_slot(ctx, slot);
  if (rc) return rc;
  rc = enqueue_frame(ctx, slot, dev_frames);
  if (rc) return rc;
  ++ctx->seq;
  return STITCH_B200_OK;
}

int stitch_b200_fork(stitch_b200_ctx* h) {
  Ctx* ctx = h->c.get();
  CUDA_TRY(cudaSetDevice(ctx->device));
  return fork_api_stream(ctx);
}

int stitch_b200_join(stitch_b200_ctx* h) {
  Ctx* ctx = h->c.get();
  CUDA_TRY(cudaSetDevice(ctx->device));
  return join_api_stream(ctx);
}

int stitch_b200_profile_frame(stitch_b200_ctx* h, const uint8_t* const* dev_frames, int max_ops,
                              int* kinds, float* ms) {
  Ctx* ctx = h->c.get();
  CUDA_TRY(cudaSetDevice(ctx->device));
  // eager run on slot 0 after draining the pipeline
  for (int sl = 0; sl < ctx->n_slots; ++sl) {
    int rc = retire_slot(ctx, sl);
    if (rc) return -rc;
  }
  for (int sl = 0; sl < ctx->n_slots; ++sl) CUDA_TRY(cudaStreamSynchronize(ctx->slot[sl].cs));
  CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  CUDA_TRY(cudaStreamSynchronize(ctx->d2h));
  int rc = set_frame_pointers(ctx, 0, dev_frames);
  if (rc) return -rc;
  CUDA_TRY(cudaStreamSynchronize(ctx->slot[0].cs));
  ctx->last_slot = 0;
  std::vector<cudaEvent_t> evs;
  std::vector<int> ks;
  cudaStream_t s = ctx->stream;
  for (const Op& op : ctx->plan) {
    if (op.kind == OP_EVENT) continue;
    cudaEvent_t a, b;
    CUDA_TRY(cudaEventCreate(&a));
    CUDA_TRY(cudaEventCreate(&b));
    CUDA_TRY(cudaEventRecord(a, s));
    const int n = enqueue_op(ctx, op, s);
    CUDA_TRY(cudaEventRecord(b, s));
    if (n == 0) {
      cudaEventDestroy(a);
      cudaEventDestroy(b);
      continue;
    }
    evs.push_back(a);
    evs.push_back(b);
    ks.push_back(static_cast<int>(op.kind));
  }
  cudaError_t e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaGetLastError();
  const int n = static_cast<int>(ks.size());
  for (int i = 0; i < n; ++i) {
    float t = 0;
    if (e == cudaSuccess) cudaEventElapsedTime(&t, evs[2 * i], evs[2 * i + 1]);
    if (i < max_ops) {
      kinds[i] = ks[i];
      ms[i] = t;
    }
  }
  for (auto& x : evs) cudaEventDestroy(x);
  if (e != cudaSuccess) return -fail(STITCH_B200_CudaError, cudaGetErrorString(e));
  return n;
}

int stitch_b200_device_pano(const stitch_b200_ctx* h, uint8_t** rgb, uint8_t** mask) {
  const Ctx* ctx = h->c.get();
  if (rgb) *rgb = ctx->d_out_rgb[ctx->last_slot];
  if (mask) *mask = ctx->d_out_mask[ctx->last_slot];
  return STITCH_B200_OK;
}

void* stitch_b200_stream(const stitch_b200_ctx* h) { return h->c->stream; }

int stitch_b200_synchronize(stitch_b200_ctx* h) { return sync_all(h->c.get()); }

int stitch_b200_launches_per_frame(const stitch_b200_ctx* h) { return h->c->launches; }

void* stitch_b200_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) return nullptr;
  return p;
}

void stitch_b200_host_free(void* p) { cudaFreeHost(p); }

int stitch_b200_debug_copy_pool(int workers, int rounds, size_t bytes) {
  // host only (no device): back-to-back batches of varying sizes through one
  // pool, every destination byte checked after each batch
  CopyPool pool(workers);
  std::vector<unsigned char> src(bytes), dst(bytes);
  for (int r = 0; r < rounds; ++r) {
    const size_t n = bytes - (static_cast<size_t>(r) * 7919u) % (bytes / 2 + 1);
    for (size_t i = 0; i < n; i += 4096) src[i] = static_cast<unsigned char>(r + i / 4096);
    const size_t half = n / 2;
    pool.run({{dst.data(), src.data(), half}, {dst.data() + half, src.data() + half, n - half}});
    if (std::memcmp(dst.data(), src.data(), n) != 0)
      return fail(STITCH_B200_InputMismatch, "copy pool produced wrong bytes");
  }
  return STITCH_B200_OK;
}

int stitch_b200_host_register(void* p, size_t bytes) {
  CUDA_TRY(cudaHostRegister(p, bytes, cudaHostRegisterDefault));
  return STITCH_B200_OK;
}

int stitch_b200_host_unregister(void* p) {
  CUDA_TRY(cudaHostUnregister(p));
  return STITCH_B200_OK;
}

void* stitch_b200_device_alloc(int device, size_t bytes) {
  void* p = nullptr;
  if (cudaSetDevice(device) != cudaSuccess) return nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
  return p;
}

void stitch_b200_device_free(void* p) { cudaFree(p); }

int stitch_b200_memcpy_h2d(void* dst, const void* src, size_t bytes) {
  CUDA_TRY(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
  return STITCH_B200_OK;
}

int stitch_b200_memcpy_d2h(void* dst, const void* src, size_t bytes) {
  CUDA_TRY(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
  return STITCH_B200_OK;
}

int stitch_b200_debug_crop(stitch_b200_ctx* h, int k, int side, int corrected, uint8_t* rgb,
                           uint8_t* mask) {
  Ctx* ctx = h->c.get();
  if (k < 0 || k >= ctx->hg.n_pairs || side < 0 || side > 1)
    return fail(STITCH_B200_ConfigurationError, "bad pair/side");
  if (int rc_ = sync_all(ctx)) return rc_;
  const PairDesc& p = ctx->slot[ctx->last_slot].hg.pairs[k];
  std::vector<uchar4> buf(static_cast<size_t>(p.w) * p.h);
  CUDA_TRY(cudaMemcpy(buf.data(), corrected ? p.crop_cor[side] : p.crop_raw[side],
                      buf.size() * sizeof(uchar4), cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < buf.size(); ++i) {
    rgb[3 * i + 0] = buf[i].x;
    rgb[3 * i + 1] = buf[i].y;
    rgb[3 * i + 2] = buf[i].z;
    mask[i] = buf[i].w;
  }
  return STITCH_B200_OK;
}

int stitch_b200_debug_flow(stitch_b200_ctx* h, int k, int dir, float* u, float* v) {
  Ctx* ctx = h->c.get();
  if (k < 0 || k >= ctx->hg.n_pairs || dir < 0 || dir > 1)
    return fail(STITCH_B200_ConfigurationError, "bad pair/dir");
  if (int rc_ = sync_all(ctx)) return rc_;
  const PairDesc& p = ctx->slot[ctx->last_slot].hg.pairs[k];
  const size_t n = static_cast<size_t>(p.w) * p.h;
  std::vector<float2> uv(n);
  CUDA_TRY(cudaMemcpy(uv.data(), p.flow_uv[dir], n * sizeof(float2), cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < n; ++i) {
    u[i] = uv[i].x;
    v[i] = uv[i].y;
  }
  // dense_flow's final zeroing where either crop is invalid (flow.cpp:178-185)
  // is applied by the flow's consumer (fused_pixel) instead of being written
  // into the plane; apply it here so the readback is the reference's field
  std::vector<uchar4> ca(n), cb(n);
  CUDA_TRY(cudaMemcpy(ca.data(), p.crop_cor[0], n * sizeof(uchar4), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(cb.data(), p.crop_cor[1], n * sizeof(uchar4), cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < n; ++i)
    if (!ca[i].w || !cb[i].w) u[i] = v[i] = 0.0f;
  return STITCH_B200_OK;
}

int stitch_b200_debug_prebalance(stitch_b200_ctx* h, uint8_t* rgb, uint8_t* mask) {
  Ctx* ctx = h->c.get();
  if (int rc_ = sync_all(ctx)) return rc_;
  std::vector<uchar4> buf(static_cast<size_t>(ctx->n_px));
  CUDA_TRY(cudaMemcpy(buf.data(), ctx->slot[ctx->last_slot].d_pano, buf.size() * sizeof(uchar4),
                      cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < buf.size(); ++i) {
    rgb[3 * i + 0] = buf[i].x;
    rgb[3 * i + 1] = buf[i].y;
    rgb[3 * i + 2] = buf[i].z;
    mask[i] = buf[i].w;
  }
  return STITCH_B200_OK;
}

int stitch_b200_debug_warp_view(stitch_b200_ctx* h, int view, const uint8_t* host_frame,
                                uint8_t* rgb, uint8_t* mask) {
  Ctx* ctx = h->c.get();
  if (view < 0 || view >= ctx->hg.n_views) return fail(STITCH_B200_ConfigurationError, "bad view");
  CUDA_TRY(cudaSetDevice(ctx->device));
  if (int rc_ = sync_all(ctx)) return rc_;
  std::uint8_t *df = nullptr, *dr = nullptr, *dm = nullptr;
  uchar4* dq = nullptr;
  const size_t n = static_cast<size_t>(ctx->n_px);
  const long long vpx = static_cast<long long>(ctx->hg.views[view].width) * ctx->hg.views[view].height;
  CUDA_TRY(cudaMalloc(&df, ctx->frame_bytes[view]));
  CUDA_TRY(cudaMalloc(&dq, vpx * sizeof(uchar4)));
  CUDA_TRY(cudaMalloc(&dr, n * 3));
  CUDA_TRY(cudaMalloc(&dm, n));
  CUDA_TRY(cudaMemcpy(df, host_frame, ctx->frame_bytes[view], cudaMemcpyHostToDevice));
  launch_expand_one(df, dq, vpx, ctx->stream);
  launch_warp_view(ctx->slot[0].dg, view, dq, dr, dm, ctx->stream);
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e == cudaSuccess) e = cudaMemcpy(rgb, dr, n * 3, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(mask, dm, n, cudaMemcpyDeviceToHost);
  cudaFree(df);
  cudaFree(dq);
  cudaFree(dr);
  cudaFree(dm);
  if (e != cudaSuccess) return fail(STITCH_B200_CudaError, cudaGetErrorString(e));
  return STITCH_B200_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// quality metrics (metrics.cpp:9-155) on the device
// ---------------------------------------------------------------------------
static int psnr_from_parts(unsigned long long sse, unsigned long long n, double* out) {
  if (n == 0) return fail(STITCH_B200_EmptyRegion, "no jointly valid pixel");
  const double mse = static_cast<double>(sse) / (3.0 * static_cast<double>(n));
  *out = mse == 0.0 ? std::numeric_limits<double>::infinity()
                    : 10.0 * std::log10(255.0 * 255.0 / mse);
  return STITCH_B200_OK;
}

static int ssim_from_parts(double sum, long long n, double* out) {
  if (n == 0) return fail(STITCH_B200_EmptyRegion, "no fully valid SSIM window");
  *out = sum / static_cast<double>(n);
  return STITCH_B200_OK;
}

namespace {
struct PackedPair {
  uchar4* a = nullptr;
  uchar4* b = nullptr;
};

// caller holds ws.mu
int pack_pair(MetricsWorkspace& ws, int w, int h, const uint8_t* a_rgb, const uint8_t* a_mask,
              const uint8_t* b_rgb, const uint8_t* b_mask, PackedPair& pp) {
  if (w <= 0 || h <= 0 || !a_rgb || !b_rgb)
    return fail(STITCH_B200_ConfigurationError, "bad frame arguments");
  const int n = w * h;
  CUDA_TRY(gpu_pack_rgba(ws, 0, a_rgb, a_mask, n, &pp.a, ws.s));
  CUDA_TRY(gpu_pack_rgba(ws, 1, b_rgb, b_mask, n, &pp.b, ws.s));
  return STITCH_B200_OK;
}
}  // namespace

int stitch_b200_psnr(int width, int height, const uint8_t* a_rgb, const uint8_t* a_mask,
                     const uint8_t* b_rgb, const uint8_t* b_mask, double* out) {
  MetricsWorkspace& ws = metrics_workspace();
  std::lock_guard<std::mutex> lk(ws.mu);
  PackedPair pp;
  int rc = pack_pair(ws, width, height, a_rgb, a_mask, b_rgb, b_mask, pp);
  if (rc) return rc;
  unsigned long long sse = 0, n = 0;
  CUDA_TRY(gpu_psnr_parts(ws, pp.a, pp.b, width * height, &sse, &n, ws.s));
  return psnr_from_parts(sse, n, out);
}

int stitch_b200_ssim(int width, int height, const uint8_t* a_rgb, const uint8_t* a_mask,
                     const uint8_t* b_rgb, const uint8_t* b_mask, double* out) {
  if (width < 11 || height < 11) return fail(STITCH_B200_TooSmall, "ssim needs >= 11x11");
  MetricsWorkspace& ws = metrics_workspace();
  std::lock_guard<std::mutex> lk(ws.mu);
  PackedPair pp;
  int rc = pack_pair(ws, width, height, a_rgb, a_mask, b_rgb, b_mask, pp);
  if (rc) return rc;
  double sum = 0.0;
  long long n = 0;
  CUDA_TRY(gpu_ssim_parts(ws, pp.a, pp.b, width, height, &sum, &n, ws.s));
  return ssim_from_parts(sum, n, out);
}

int stitch_b200_pair_quality(stitch_b200_ctx* h, int k, double out[3]) {
  Ctx* ctx = h->c.get();
  if (k < 0 || k >= ctx->hg.n_pairs) return fail(STITCH_B200_ConfigurationError, "bad pair index");
  if (int rc_ = sync_all(ctx)) return rc_;
  const PairDesc& p = ctx->slot[ctx->last_slot].hg.pairs[k];
  const int n = p.w * p.h;
  CUDA_TRY(cudaSetDevice(ctx->device));
  MetricsWorkspace& ws = metrics_workspace();
  std::lock_guard<std::mutex> lk(ws.mu);
  unsigned long long sse = 0, cnt = 0;
  CUDA_TRY(gpu_psnr_parts(ws, p.crop_cor[0], p.crop_raw[0], n, &sse, &cnt, ctx->stream));
  int rc = psnr_from_parts(sse, cnt, &out[0]);
  if (rc) return rc;
  CUDA_TRY(gpu_psnr_parts(ws, p.crop_cor[0], p.crop_cor[1], n, &sse, &cnt, ctx->stream));
  rc = psnr_from_parts(sse, cnt, &out[1]);
  if (rc) return rc;
  if (p.w < 11 || p.h < 11) return fail(STITCH_B200_TooSmall, "ssim needs >= 11x11");
  double sum = 0.0;
  long long wn = 0;
  CUDA_TRY(gpu_ssim_parts(ws, p.crop_cor[0], p.crop_cor[1], p.w, p.h, &sum, &wn, ctx->stream));
  return ssim_from_parts(sum, wn, &out[2]);
}

// ---------------------------------------------------------------------------
// feature-path diagnostics
// ---------------------------------------------------------------------------
int stitch_b200_debug_detect(int width, int height, const uint8_t* rgb, const int region[4],
                             double threshold, int max_kp, double* kp, float* desc) {
  if (width <= 0 || height <= 0 || !rgb || !region)
    return -fail(STITCH_B200_ConfigurationError, "bad frame arguments");
  if (region[2] - region[0] < 32 || region[3] - region[1] < 32)
    return -fail(STITCH_B200_RegionTooSmall, "detection region must be at least 32x32");
  const size_t n = static_cast<size_t>(width) * height * 3;
  void* d = nullptr;
  if (cudaMalloc(&d, n) != cudaSuccess) return -fail(STITCH_B200_CudaError, "cudaMalloc");
  std::unique_ptr<void, cudaError_t (*)(void*)> guard(d, cudaFree);
  if (cudaMemcpy(d, rgb, n, cudaMemcpyHostToDevice) != cudaSuccess)
    return -fail(STITCH_B200_CudaError, "cudaMemcpy");
  FeatView fv;
  std::vector<FeatPoint> kps;
  std::vector<float> ds;
  cudaError_t e = fv.build(static_cast<const std::uint8_t*>(d), width, height, nullptr);
  if (e == cudaSuccess)
    e = fv.detect_describe(region[0], region[1], region[2], region[3], threshold, kps, ds, nullptr);
  if (e != cudaSuccess) return -fail(STITCH_B200_CudaError, cudaGetErrorString(e));
  const int m = std::min<int>(max_kp, static_cast<int>(kps.size()));
  for (int i = 0; i < m; ++i) {
    kp[4 * i + 0] = kps[i].x;
    kp[4 * i + 1] = kps[i].y;
    kp[4 * i + 2] = kps[i].scale;
    kp[4 * i + 3] = kps[i].response;
    std::memcpy(desc + 64 * static_cast<size_t>(i), ds.data() + 64 * static_cast<size_t>(i),
                64 * sizeof(float));
  }
  return static_cast<int>(kps.size());
}

int stitch_b200_debug_tone_curves(int n, const int* m1, const int* m2, double gamma_dark,
                                  double gamma_bright, int target_black, int target_white,
                                  uint8_t* out) {
  if (n < 0) return fail(STITCH_B200_ConfigurationError, "negative curve count");
  if (n == 0) return STITCH_B200_OK;
  int *d1 = nullptr, *d2 = nullptr;
  uint8_t* dout = nullptr;
  const size_t ib = sizeof(int) * static_cast<size_t>(n), ob = 256 * static_cast<size_t>(n);
  cudaError_t e = cudaMalloc(&d1, ib);
  if (e == cudaSuccess) e = cudaMalloc(&d2, ib);
  if (e == cudaSuccess) e = cudaMalloc(&dout, ob);
  if (e == cudaSuccess) e = cudaMemcpy(d1, m1, ib, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d2, m2, ib, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    stitch_b200_dev::launch_debug_tone_curves(n, d1, d2, gamma_dark, gamma_bright, target_black,
                                              target_white, dout, 0);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(out, dout, ob, cudaMemcpyDeviceToHost);
  cudaFree(d1);
  cudaFree(d2);
  cudaFree(dout);
  if (e != cudaSuccess) return fail(STITCH_B200_CudaError, cudaGetErrorString(e));
  return STITCH_B200_OK;
}

int stitch_b200_debug_match(const float* da, int na, const float* db, int nb, double ratio,
                            int* best_b, double* best_dist, int* best_a) {
  std::vector<float> a(da, da + 64 * static_cast<size_t>(na)), b(db, db + 64 * static_cast<size_t>(nb));
  std::vector<int> bb, ba;
  std::vector<double> bd;
  CUDA_TRY(feat_match(a, b, na, nb, ratio, bb, bd, ba, nullptr));
  std::copy(bb.begin(), bb.end(), best_b);
  std::copy(bd.begin(), bd.end(), best_dist);
  std::copy(ba.begin(), ba.end(), best_a);
  return STITCH_B200_OK;
}
