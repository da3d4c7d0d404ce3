#!/usr/bin/env python
"""Benchmark of the per-frame stitching hot path (BASELINE.json metric).

Workload (BASELINE.json configs[1]): 4 synthetic 1920x1080 RGB cameras, coarse
homographies (3 % focal perturbation, strip rig), overlap optical flow, 3D-M
colour transfer and global balancing -> one panorama per step.  One panorama
stream per GPU; at N GPUs each rank runs its own stream (independent streams,
no collective on the frame path; "scaling": "weak").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

value  : aggregate panorama frames/s with the input frames resident in HBM
         (stitch_b200_process_device_async, one frame per pipeline slot in flight over the
         context's pipeline slots), CUDA-event timed on the context's API
         stream around a fork and a join, max over ranks.
e2e    : the same metric through the reference-facing C-ABI calls with
         pinned HOST frames (stitch_b200_submit / stitch_b200_wait, four in
         flight): H2D of every camera frame + D2H of the balanced panorama
         (RGB + mask) inside the timed region, max over ranks; the
         synchronous stitch_b200_process is reported as sync_process_value.
--impl reference : the reference's CPU path on the box's host cores, rank 0
         only.  c1 (2 views, the reference's own rig) runs THE REFERENCE
         ITSELF: the unmodified sources compiled into oracle/_ref (Eigen-subset
         shim, oracle/ref/Makefile), kind "reference".  c2-c5 need 4-8 views,
         which the reference rejects ("pipeline supports 2 or 3 views",
         pipeline.cpp:24-29), so they run the oracle port (oracle/liboracle.so,
         bit-exact with the reference on <= 3 views, tests/test_ref_pin.py),
         kind "port", with the reference/port speed ratio measured on c1 in
         the same run.

--gpus N : N ranks, one per GPU.  Launched by torchrun (WORLD_SIZE set) or,
         when WORLD_SIZE is unset, bench.py spawns the N ranks itself
         (RANK / LOCAL_RANK / WORLD_SIZE / MASTER_*); gloo carries the barrier
         and the timing reductions -- the frame path has no collective.
--config c5 : BASELINE configs[4], 64 independent 4x1080p streams sharded
         s mod N over the ranks (strong scaling: the total is fixed).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "stitched panorama frames/s & p50 ms/frame, 4x1080p cams; achieved HBM GB/s"
UNIT = "frames/s"

WORKLOADS = {
    # BASELINE.json configs[1] (headline)
    "c2": dict(views=4, width=1920, height=1080, focal_scale=1.03,
               desc="4 cameras 1920x1080 RGB, coarse homographies + overlap optical flow"),
    # BASELINE.json configs[0] (reference CPU-runnable case)
    "c1": dict(views=2, width=640, height=480, focal_scale=1.0,
               desc="2 synthetic 640x480 RGB camera streams, one overlap, fixed homography"),
    # BASELINE.json configs[2] (extension: cylindrical canvas, ring chain)
    "c3": dict(views=6, width=1920, height=1080, focal_scale=1.0, rig="ring",
               desc="6-camera 360-degree ring at 1080p, 3D-M temporal colour transfer, "
                    "piecewise global balancing"),
    # BASELINE.json configs[3]
    "c4": dict(views=8, width=3840, height=2160, focal_scale=1.03,
               desc="8 cameras 3840x2160 RGB single panorama stream"),
}
# BASELINE.json configs[4]: 64 independent 4x1080p streams sharded over the
# GPUs (s mod N) -- the c2 workload with a fixed total stream count
WORKLOADS["c5"] = dict(WORKLOADS["c2"], total_streams=64,
                       desc="64 independent 4x1080p panorama streams sharded over the GPUs")


def scene_params(wl, seed):
    """The synthetic scene of a workload (SynthSpec terms, synth.hpp:31-44)."""
    nv = wl["views"]
    return dict(seed=seed, views=nv, width=wl["width"], height=wl["height"],
                focal_scale=wl["focal_scale"],
                casts=[(1.0, 1.0, 1.0) if v % 2 == 0 else (0.88, 1.0, 1.08) for v in range(nv)],
                flicker=[dict(frame=5, view=nv - 1, gains=(1.15, 1.1, 0.95))],
                obj=dict(enabled=True, half_size=0.08 * wl["width"] * 500 / (0.9 * wl["width"]),
                         velocity=(4.0, 1.0)))


def build_scene(wl, seed):
    import paper_2308_09209_b200 as pb

    p = scene_params(wl, seed)
    spec = pb.SynthSpec(seed=seed, views=p["views"], frames=300, width=p["width"],
                        height=p["height"], overlap_fraction=0.3,
                        perturb_focal_scale=p["focal_scale"], rig=wl.get("rig", "auto"))
    spec.color_casts = p["casts"]
    spec.flicker = [pb.FlickerEvent(**f) for f in p["flicker"]]
    spec.object = pb.ParallaxObject(enabled=True, half_size=p["obj"]["half_size"],
                                    velocity=p["obj"]["velocity"])
    return pb.SynthScene(spec)


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md "clocks DURING the timed region")
# ---------------------------------------------------------------------------
REASON_BITS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
    0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
    0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


class ClockSampler:
    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples = []
        self.proc = None
        self.thread = None
        self.active = False

    def start(self):
        cmd = ["nvidia-smi", "-i", str(self.gpu),
               "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
               "--format=csv,noheader,nounits", "-lms", "100"]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 3:
                continue
            try:
                sm, smax = float(parts[0]), float(parts[1])
                reasons = int(parts[2], 16)
            except ValueError:
                continue
            self.samples.append((time.perf_counter(), self.active, sm, smax, reasons))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        under = [s for s in self.samples if s[1]] or self.samples
        if not under:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = set()
        for s in under:
            for bit, name in REASON_BITS.items():
                if s[4] & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[2] for s in under),
                "sm_max_mhz": max(s[3] for s in under), "reasons": sorted(reasons),
                "samples": len(under)}


# ---------------------------------------------------------------------------
# per-kernel algorithmic bytes / flops
# ---------------------------------------------------------------------------
def pair_levels(p, levels=4):
    w, h = p.bounds[2] - p.bounds[0], p.bounds[3] - p.bounds[1]
    if w < 16 or h < 16:
        return []
    dims = [(w, h)]
    for _ in range(1, levels):
        if dims[-1][0] < 16 or dims[-1][1] < 16:
            break
        dims.append((max(1, dims[-1][0] // 2), max(1, dims[-1][1] // 2)))
    return dims


def kernel_model(state, wl, sweeps=10, warps=5, lin_levels=None):
    """Algorithmic HBM bytes (and FP32 flops for the flow) per frame, per
    kernel family.  lin_levels: how many of the finest
    levels run the separate linearisation launch (the coarser ones fuse it
    into their first Jacobi segment); None = all."""
    pairs = state.pairs
    o = [(p.bounds[2] - p.bounds[0]) * (p.bounds[3] - p.bounds[1]) for p in pairs]
    P = state.canvas_width * state.canvas_height
    in_px = wl["views"] * wl["width"] * wl["height"]
    lv = [pair_levels(p) for p in pairs]
    flow_px = 2 * sum(a * b for dims in lv for a, b in dims)  # both directions, all levels
    nl = max((len(d) for d in lv), default=0) if lin_levels is None else lin_levels
    lin_px = 2 * sum(a * b for dims in lv for a, b in dims[:nl])  # separately linearised
    fused_px = flow_px - lin_px
    coarse_px = 2 * sum(a * b for dims in lv for a, b in dims[:-1])  # finer levels (upsampled u0)
    segs = int(os.environ.get("STITCH_B200_HS_SEGS", "2"))
    elin = os.environ.get("STITCH_B200_HS_ELIN", "1") != "0"
    return {
        # RGB8 read, RGBA8 write
        "expand_rgba": dict(bytes=7 * in_px),
        # each crop pixel: one RGBA source pixel read (4 B), uchar4 write; both sides
        "crop_warp": dict(bytes=sum(2 * (4 + 4) * n for n in o)),
        # two uchar4 crops read
        "pair_color": dict(bytes=sum(8 * n for n in o)),
        # raw crops read, corrected crops + luma written
        "flow_prepare": dict(bytes=sum(2 * (4 + 4 + 4) * n for n in o)),
        # per warp iteration and pixel: u0 (8) + a (4) + b (4) read, 4 constant planes
        # (16) written; + u0 materialised (8) on each level's first warp
        "hs_linearize": dict(bytes=warps * 32 * lin_px + 8 * lin_px),
        # per segment and pixel: state (8) + constants (16) read, state (8) written.
        # On the fused (coarse) levels the first warp iteration's first segment
        # linearises in its prologue (+8: a, b read; constants written instead of
        # read), and the last segment of warp iterations 1-4 linearises the next
        # one in its epilogue (+24: a, b read, next constants written); with
        # STITCH_B200_HS_ELIN=0 every warp iteration uses the prologue
        "hs_sweeps": dict(bytes=warps * segs * 32 * flow_px + (
            (8 + 24 * (warps - 1)) * fused_px if elin else warps * 8 * fused_px),
                          flops=warps * sweeps * 17 * flow_px),
        # per canvas pixel one RGBA source pixel read + uchar4 write; overlap pixels add
        # raw crops (8) + corrected crop samples (8) + flows (16) + weight (4)
        "canvas_balance": dict(bytes=8 * P + 36 * sum(o)),
        # uchar4 pano read, RGB + mask write
        "tone": dict(bytes=8 * P),
        "_coarse_px": coarse_px,
    }


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def run_b200(args, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_2308_09209_b200 as pb
    from paper_2308_09209_b200 import _abi, sharding

    lib = _abi.load()
    # one rank per GPU; more ranks than visible GPUs (a functional run of the
    # multi-rank path on one box) share devices round-robin and say so
    n_dev = max(1, torch.cuda.device_count())
    device = local_rank % n_dev
    torch.cuda.set_device(device)
    wl = WORKLOADS[args.config]
    # streams: one per GPU (weak scaling) unless a fixed total is set (c5)
    fixed_total = args.total_streams or wl.get("total_streams", 0)
    total_streams = fixed_total if fixed_total else world * args.streams_per_gpu
    my_streams = sharding.stream_assignment(total_streams, world, rank)
    ns = len(my_streams)
    sc = build_scene(wl, seed=1 + rank)
    cfg = sc.config()  # refinement on, like the reference's default (pipeline.hpp:24)
    cfg.device = device
    nv = wl["views"]
    F = args.frame_sets
    threads = max(1, cpu_cores() // max(1, world))
    frame_bytes = wl["width"] * wl["height"] * 3
    # pre-render F frame sets, stage them in pinned host memory and in HBM
    # (shared read-only by this rank's streams)
    host_sets, dev_sets = [], []
    for t in range(F):
        hs, ds = [], []
        for v in range(nv):
            img = sc.render_view(v, t, threads).data
            hp = lib.stitch_b200_host_alloc(frame_bytes)
            C.memmove(hp, img.ctypes.data, frame_bytes)
            dp = lib.stitch_b200_device_alloc(device, frame_bytes)
            pb.pipeline.check(lib.stitch_b200_memcpy_h2d(dp, hp, frame_bytes))
            hs.append(hp)
            ds.append(dp)
        host_sets.append((C.c_void_p * nv)(*hs))
        dev_sets.append((C.c_void_p * nv)(*ds))
    # initialize() on the first frames (feature refinement of the coarse
    # homographies, pipeline.cpp:241-255) -- init time, outside every timing
    first = [sc.render_view(v, 0, threads) for v in range(nv)]
    states = [pb.initialize(cfg, first) for _ in range(ns)]
    state = states[0]
    hs_ = [st.handle for st in states]
    P = state.canvas_width * state.canvas_height
    out_rgb = lib.stitch_b200_host_alloc(P * 3)
    out_mask = lib.stitch_b200_host_alloc(P)
    cstreams = [torch.cuda.ExternalStream(lib.stitch_b200_stream(h), device=device)
                for h in hs_]
    main = torch.cuda.current_stream()
    launches = state.launches_per_frame()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def step_all(i):
        # pipelined device-resident frames (two slots per context, ordered
        # only where the temporal state requires it); joined below
        for j, h in enumerate(hs_):
            pb.pipeline.check(lib.stitch_b200_process_device_async(h, dev_sets[(i + j) % F]))

    clocks = ClockSampler(device)
    clocks.start()
    # ---- warm-up ----
    for i in range(args.warmup):
        step_all(i)
    for h in hs_:
        pb.pipeline.check(lib.stitch_b200_synchronize(h))
    torch.cuda.synchronize()
    # ---- timed: device-resident inputs; all streams of this rank ----
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    clocks.active = True
    e0.record(main)
    for cs in cstreams:
        cs.wait_event(e0)
    for h in hs_:
        pb.pipeline.check(lib.stitch_b200_fork(h))
    for i in range(args.steps):
        step_all(i)
    for h in hs_:
        pb.pipeline.check(lib.stitch_b200_join(h))
    for cs in cstreams:
        ev = torch.cuda.Event()
        ev.record(cs)
        main.wait_event(ev)
    e1.record(main)
    torch.cuda.synchronize()
    clocks.active = False
    barrier()
    elapsed_s = e0.elapsed_time(e1) / 1e3
    max_s = sharding.max_over_ranks(elapsed_s)
    frames_total = sharding.sum_over_ranks(ns * args.steps)
    value = frames_total / max_s
    ms_per_step = max_s * 1e3 / args.steps

    # ---- per-frame latency distribution of one stream (p50) ----
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(min(args.steps, 200))]
    for i, (a, b) in enumerate(evs):
        a.record(cstreams[0])
        pb.pipeline.check(lib.stitch_b200_process_device(hs_[0], dev_sets[i % F], None))
        b.record(cstreams[0])
    torch.cuda.synchronize()
    p50 = statistics.median(a.elapsed_time(b) for a, b in evs)

    # ---- e2e: the C-ABI host-buffer path, pipelined (stitch_b200_submit /
    # stitch_b200_wait, two frames in flight): H2D of every frame's camera
    # images and D2H of every balanced panorama + mask inside the timed region
    # a fixed e2e sample (not --steps): long enough that the 4-deep pipeline
    # fill is negligible
    e2e_steps = max(1, args.e2e_steps)
    depth = lib.stitch_b200_slots(hs_[0])  # frames in flight = the context's slots
    outs = [(lib.stitch_b200_host_alloc(P * 3), lib.stitch_b200_host_alloc(P))
            for _ in range(depth)]
    tk = C.c_longlong()

    def e2e_run(n):
        tickets = []
        for i in range(n):
            o = outs[i % depth]
            pb.pipeline.check(lib.stitch_b200_submit(hs_[0], host_sets[i % F], o[0], o[1],
                                                     C.byref(tk)))
            tickets.append(tk.value)
            if i >= depth - 1:
                pb.pipeline.check(lib.stitch_b200_wait(hs_[0], tickets[i - depth + 1], None))
        for t in tickets[max(0, n - depth + 1):]:
            pb.pipeline.check(lib.stitch_b200_wait(hs_[0], t, None))

    e2e_run(min(args.warmup, 3) + 1)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_run(e2e_steps)
    e2e_s = sharding.max_over_ranks(time.perf_counter() - t0)
    e2e_value = world * e2e_steps / e2e_s
    # the same with PAGEABLE host buffers (the reference's std::vector frames,
    # frame.hpp:17-57): the context stages them through its pinned ring
    pg_in = [[np.empty(frame_bytes, np.uint8) for _ in range(nv)] for _ in range(F)]
    for t in range(F):
        for v in range(nv):
            C.memmove(pg_in[t][v].ctypes.data, host_sets[t][v], frame_bytes)
    pg_in_ptrs = [(C.c_void_p * nv)(*[a.ctypes.data for a in pg_in[t]]) for t in range(F)]
    pg_out = [(np.empty(P * 3, np.uint8), np.empty(P, np.uint8)) for _ in range(depth)]

    def e2e_run_pageable(n):
        tickets = []
        for i in range(n):
            o = pg_out[i % depth]
            pb.pipeline.check(lib.stitch_b200_submit(hs_[0], pg_in_ptrs[i % F], o[0].ctypes.data,
                                                     o[1].ctypes.data, C.byref(tk)))
            tickets.append(tk.value)
            if i >= depth - 1:
                pb.pipeline.check(lib.stitch_b200_wait(hs_[0], tickets[i - depth + 1], None))
        for t in tickets[max(0, n - depth + 1):]:
            pb.pipeline.check(lib.stitch_b200_wait(hs_[0], t, None))

    e2e_run_pageable(min(args.warmup, 3) + 1)
    barrier()
    t0 = time.perf_counter()
    e2e_run_pageable(e2e_steps)
    e2e_pg_s = sharding.max_over_ranks(time.perf_counter() - t0)
    e2e_pageable = world * e2e_steps / e2e_pg_s
    # the same through the synchronous call (reference semantics, no overlap)
    t0 = time.perf_counter()
    for i in range(min(e2e_steps, 50)):
        pb.pipeline.check(lib.stitch_b200_process(hs_[0], host_sets[i % F], out_rgb, out_mask,
                                                  None))
    e2e_sync_s = sharding.max_over_ranks(time.perf_counter() - t0)
    e2e_sync = world * min(e2e_steps, 50) / e2e_sync_s
    # ... and with pageable buffers: the drop-in binding's call (INTEGRATION.md:
    # process_frame_b200 hands the reference's std::vector frames to
    # stitch_b200_process)
    t0 = time.perf_counter()
    for i in range(min(e2e_steps, 50)):
        pb.pipeline.check(lib.stitch_b200_process(hs_[0], pg_in_ptrs[i % F],
                                                  pg_out[0][0].ctypes.data,
                                                  pg_out[0][1].ctypes.data, None))
    e2e_sync_pg_s = sharding.max_over_ranks(time.perf_counter() - t0)
    e2e_sync_pg = world * min(e2e_steps, 50) / e2e_sync_pg_s

    # ---- per-kernel profile (eager plan, CUDA events around each launch) ----
    n_ops = 4096
    kinds = (C.c_int * n_ops)()
    ms = (C.c_float * n_ops)()
    per_kind = {}
    prof_frames = 5
    for i in range(prof_frames):
        n = lib.stitch_b200_profile_frame(hs_[0], dev_sets[i % F], n_ops, kinds, ms)
        if n < 0:
            pb.pipeline.check(-n)
        for j in range(min(n, n_ops)):
            name = _abi.OP_KIND_NAMES[kinds[j]]
            d = per_kind.setdefault(name, [0.0, 0])
            d[0] += ms[j] / prof_frames
            d[1] += 1 if i == 0 else 0
    clocks.stop()

    peak, peak_kind = load_peaks()
    lin_launches = per_kind.get("hs_linearize", [0.0, 0])[1]
    model = kernel_model(state, wl, lin_levels=lin_launches // 5)
    total_kernel_ms = sum(v[0] for v in per_kind.values())
    clk = clocks.summary()
    fp32_peak = 148 * 128 * (clk.get("sm_mhz") or 1965.0) * 1e6 / 1e12  # add/mul, no FMA
    kernels = {}
    for name, (t_ms, count) in sorted(per_kind.items(), key=lambda kv: -kv[1][0]):
        mdl = model.get(name, {})
        k = {"ms_per_frame": round(t_ms, 4), "launches_per_frame": count,
             "share": round(t_ms / total_kernel_ms, 4) if total_kernel_ms else None}
        if "bytes" in mdl and t_ms > 0:
            k["alg_bytes_per_frame"] = mdl["bytes"]
            k["hbm_gbs"] = round(mdl["bytes"] / (t_ms * 1e-3) / 1e9, 1)
            k["hbm_frac"] = round(k["hbm_gbs"] / peak, 4)
        if "flops" in mdl and t_ms > 0:
            k["fp32_tflops"] = round(mdl["flops"] / (t_ms * 1e-3) / 1e12, 3)
            k["fp32_frac"] = round(k["fp32_tflops"] / fp32_peak, 4)
        kernels[name] = k
    dominant = max(per_kind, key=lambda n: per_kind[n][0])
    dk = kernels[dominant]
    # ncu DRAM bytes per launch of the dominant kernel (read + write, one
    # frame's launches averaged: profiles/traffic.json from the committed
    # launch list), comparable with alg_bytes_per_launch
    traffic, traffic_src = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f).get(dominant)
        if t:
            traffic, traffic_src = int(t["dram_bytes_per_launch"]), t["source"]
    except Exception:
        pass
    launches_dom = max(1, dk["launches_per_frame"])
    roofline = {"kernel": dominant, "bound": "hbm", "achieved": dk.get("hbm_gbs"), "peak": peak,
                "unit": "GB/s", "frac": dk.get("hbm_frac"), "traffic": traffic,
                "traffic_source": traffic_src,
                "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                "alg_bytes_per_launch": (model[dominant]["bytes"] / launches_dom
                                         if dominant in model else None),
                "note": ("the dominant kernel is FP32-issue/SMEM bound (bit-exact unfused "
                         "Jacobi), see roofline_fp32; HBM-streaming kernels in hbm_kernels")}
    roofline_fp32 = None
    if "fp32_tflops" in dk:
        roofline_fp32 = {"kernel": dominant, "bound": "fp32 (add/mul issue, FMA not allowed)",
                         "achieved": dk["fp32_tflops"], "peak": round(fp32_peak, 2),
                         "unit": "TFLOP/s", "frac": dk["fp32_frac"]}
    hbm_kernels = {n: kernels[n] for n in ("tone", "expand_rgba", "canvas_balance", "crop_warp",
                                           "pair_color", "flow_prepare", "hs_linearize")
                   if n in kernels}

    result = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "p50_ms_per_frame": round(p50, 4), "higher_is_better": True,
        "scaling": "strong" if fixed_total else "weak",
        "vs_baseline": None, "dtype": "u8 (fp64 warp, fp32 flow)",
        "data": ("synthetic (procedural plane scene: the repo's SynthScene, byte-identical to "
                 "the reference's renderer on <= 3 views; seed 1+rank)"),
        "config": {"workload": wl["desc"], "config_key": args.config, "cameras": nv,
                   "camera_size": [wl["width"], wl["height"]],
                   "canvas": [state.canvas_width, state.canvas_height],
                   "pairs": [list(p.bounds) for p in state.pairs],
                   "streams_total": int(total_streams), "streams_this_rank": ns,
                   "parallelism": f"independent streams sharded over {world} GPU(s), no collective",
                   "refined_pairs": sum(1 for p in state.pairs if not p.refine_warning),
                   "gpus_visible": n_dev,
                   "oversubscribed": world > n_dev,
                   "l2": (f"inputs cycle over {F} pre-rendered frame sets "
                          f"({F * nv * frame_bytes / 1e6:.0f} MB > 126 MB L2)")},
        "e2e": {"value": round(e2e_value, 2), "unit": UNIT,
                "h2d_bytes_per_step": nv * frame_bytes, "d2h_bytes_per_step": P * 4,
                "steps": e2e_steps, "streams": 1,
                "api": f"stitch_b200_submit/stitch_b200_wait ({depth} frames in flight, pinned host)",
                "sync_process_value": round(e2e_sync, 2),
                "sync_pageable_value": round(e2e_sync_pg, 2),
                "pageable_value": round(e2e_pageable, 2),
                "pageable_api": "same calls with pageable (numpy) frames and outputs, staged "
                                "through the context's pinned ring"},
        "realtime_streams": round(value / 30.0, 1),  # sustained 30 fps streams
        "gpu_launches": launches * args.steps * ns,
        "kernels_per_frame": launches,
        "roofline": roofline,
        "roofline_fp32": roofline_fp32,
        "hbm_kernels": hbm_kernels,
        "kernels": kernels,
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(args, wl, sample_seconds=args.cpu_seconds)
    return result


# ---------------------------------------------------------------------------
# CPU arms: the reference itself (oracle/_ref) or the oracle port -- baseline
# and reference arm only, never the measured product
# ---------------------------------------------------------------------------
class CpuRunner:
    """One stream of the workload on the host: `kind` "reference" runs the
    compiled reference sources (stitch::initialize / process_frame through
    oracle/reference.py), "port" the oracle restatement (oracle/liboracle.so).
    Both initialize on the first frames with the reference's default feature
    refinement, like the B200 arm."""

    def __init__(self, wl, kind, threads, n_sets=2):
        self.kind = kind
        p = scene_params(wl, seed=1)
        if kind == "reference":
            import oracle.reference as R

            sc = R.Scene(seed=1, views=p["views"], frames=300, width=p["width"],
                         height=p["height"], casts=p["casts"], flicker=p["flicker"],
                         obj=p["obj"], focal_scale=p["focal_scale"])
            self.frames = [[sc.render(v, t) for v in range(p["views"])] for t in range(n_sets)]
            self.st = R.State(sc, R.default_opts(threads=threads), self.frames[0])
            sc.close()
        else:
            import oracle as O

            sc = build_scene(wl, seed=1)
            c = sc.config_c()
            cams = [(c.cams[v].fx, c.cams[v].fy, c.cams[v].cx, c.cams[v].cy,
                     list(c.cams[v].rotation), list(c.cams[v].translation))
                    for v in range(c.n_views)]
            sizes = [(c.width[v], c.height[v]) for v in range(c.n_views)]
            self.frames = [[sc.render_view(v, t, threads).data for v in range(p["views"])]
                           for t in range(n_sets)]
            cfg = O.make_config(c.n_views, c.reference, sizes, cams, threads=threads,
                                topology=c.topology, projection=c.projection,
                                cyl_focal=c.cyl_focal, refine=c.projection == 0,
                                seed=sc.spec.seed)
            self.st = O.OracleState(cfg, first_frames=self.frames[0])
            sc.close()

    def geometry(self):
        """canvas size, pair bounds and refined-pair count of the initialized
        state: the same values the B200 arm reports for the workload."""
        cw, ch = int(self.st.canvas[0]), int(self.st.canvas[1])
        pairs, refined = [], 0
        for k in range(self.st.n_pairs()):
            pr = self.st.pair(k)
            if self.kind == "reference":
                _, b, warn = pr
            else:
                _, _, b = pr
                warn = self.st.refine_warning(k)
            pairs.append([int(x) for x in b])
            refined += 0 if warn else 1
        return [cw, ch], pairs, refined

    def rate(self, seconds, max_frames=None, warmup=1):
        for i in range(warmup):
            self.st.process(self.frames[i % len(self.frames)])
        n, t0 = 0, time.perf_counter()
        while True:
            self.st.process(self.frames[n % len(self.frames)])
            n += 1
            el = time.perf_counter() - t0
            if el >= seconds or (max_frames and n >= max_frames):
                return n, el

    def close(self):
        self.st.close()


def reference_kind(wl):
    """The reference itself where it runs the workload (2-3 views, planar),
    else the port."""
    import oracle.reference as R

    if wl["views"] <= 3 and wl.get("rig", "auto") != "ring" and R.available():
        return "reference"
    return "port"


def cpu_baseline(args, wl, sample_seconds=15.0):
    threads = cpu_cores()
    kind = reference_kind(wl)
    r = CpuRunner(wl, kind, threads)
    n, el = r.rate(sample_seconds)
    r.close()
    src = ("oracle/_ref/libstitch_ref.so: the unmodified reference sources"
           if kind == "reference" else "oracle/liboracle.so: the reference path restated in C")
    out = {"value": round(n / el, 4), "unit": UNIT, "cores": threads, "kind": kind,
           "sample": f"{n} frames of the same workload after 1 warm-up frame "
                     f"({el:.1f} s, {src}, {threads} threads)"}
    # single-thread rate (the paper's Table-4 shaped CPU ratio), a shorter sample
    r1 = CpuRunner(wl, kind, 1)
    n1, el1 = r1.rate(sample_seconds / 3)
    r1.close()
    out["value_1_thread"] = round(n1 / el1, 4)
    out["sample_1_thread"] = f"{n1} frames, {el1:.1f} s, 1 thread"
    return out


def reference_vs_port(seconds=6.0):
    """Speed of the reference itself vs the port on c1 (both run it), so a
    port-timed reference arm can be read against the real reference."""
    import oracle.reference as R

    if not R.available():
        return None
    threads = cpu_cores()
    out = {}
    for kind in ("reference", "port"):
        r = CpuRunner(WORKLOADS["c1"], kind, threads)
        n, el = r.rate(seconds)
        r.close()
        out[kind] = round(n / el, 4)
    out["reference_over_port"] = round(out["reference"] / out["port"], 4)
    out["note"] = f"c1 frames/s on {threads} host threads, same run"
    return out


def run_reference(args):
    wl = WORKLOADS[args.config]
    threads = cpu_cores()
    kind = reference_kind(wl)
    r = CpuRunner(wl, kind, threads, n_sets=min(4, max(1, args.frame_sets)))
    budget = args.ref_budget_s
    t_w = time.perf_counter()
    for i in range(args.warmup):
        r.st.process(r.frames[i % len(r.frames)])
        if time.perf_counter() - t_w > budget / 4:
            break
    n, t0 = 0, time.perf_counter()
    for i in range(args.steps):
        r.st.process(r.frames[i % len(r.frames)])
        n += 1
        if time.perf_counter() - t0 > budget:
            break
    el = time.perf_counter() - t0
    canvas, pairs, refined = r.geometry()
    r.close()
    v = n / el
    if kind == "reference":
        what = ("oracle/_ref/libstitch_ref.so: the unmodified reference sources "
                "(stitch::initialize + process_frame), Eigen-subset shim")
    else:
        what = ("oracle/liboracle.so: the reference path restated in C, bit-exact with the "
                "reference on <= 3 views; the reference itself rejects "
                f"{wl['views']} views (pipeline.cpp:24-29)")
    res = {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": UNIT,
           "n_gpus": 0, "steps": n, "warmup": args.warmup, "ms_per_step": round(1e3 * el / n, 2),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "u8 (fp64 warp, fp32 flow)", "data": "synthetic",
           "config": {"workload": wl["desc"], "config_key": args.config,
                      "cameras": wl["views"], "camera_size": [wl["width"], wl["height"]],
                      "canvas": canvas, "pairs": pairs, "streams_total": 1,
                      "refined_pairs": refined,
                      "parallelism": f"one stream on {threads} host threads (CPU reference arm)"},
           "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": threads, "kind": kind,
                            "sample": f"{n} of {args.steps} requested frames within a "
                                      f"{budget:.0f} s budget ({what})"},
           "e2e": {"value": round(v, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    if kind == "port" and not args.no_calibration:
        res["reference_vs_port_c1"] = reference_vs_port()
    return res


def spawn_ranks(n):
    """bench.py --gpus N without torchrun: run N copies of this script as
    ranks 0..N-1 (one per GPU) and relay rank 0's output."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:],
                                      env=env, stdout=None if r == 0 else subprocess.DEVNULL))
    # a rank that fails would leave the others waiting at the barrier: stop
    # them as soon as one exits non-zero
    rcs = [None] * n
    while any(rc is None for rc in rcs):
        for i, p in enumerate(procs):
            if rcs[i] is None:
                rcs[i] = p.poll()
        if any(rc not in (None, 0) for rc in rcs):
            for i, p in enumerate(procs):
                if rcs[i] is None:
                    p.terminate()
            for i, p in enumerate(procs):
                if rcs[i] is None:
                    try:
                        rcs[i] = p.wait(timeout=30)
                    except subprocess.TimeoutExpired:
                        p.kill()
                        rcs[i] = p.wait()
            break
        time.sleep(0.2)
    return max(rcs, key=abs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--frame-sets", type=int, default=16)
    ap.add_argument("--streams-per-gpu", type=int, default=1)
    ap.add_argument("--total-streams", type=int, default=0,
                    help="fixed stream count sharded over the ranks (c5 sets 64)")
    ap.add_argument("--e2e-steps", type=int, default=200)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-budget-s", type=float, default=120.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-calibration", action="store_true",
                    help="reference arm: skip the c1 reference-vs-port speed ratio")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        if rank != 0:
            return
        print(json.dumps(run_reference(args)), flush=True)
        return
    if world > 1:
        import torch

        import datetime

        # gloo: only the barrier and the timing reductions cross ranks
        torch.distributed.init_process_group("gloo", rank=rank, world_size=world,
                                             timeout=datetime.timedelta(minutes=15))
    res = run_b200(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch

        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
