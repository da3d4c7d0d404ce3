#!/usr/bin/env python
"""Benchmark of the per-frame stitching hot path (BASELINE.json metric).

Workload (BASELINE.json configs[1]): 4 synthetic 1920x1080 RGB cameras, coarse
homographies (3 % focal perturbation, strip rig), overlap optical flow, 3D-M
colour transfer and global balancing -> one panorama per step.  One panorama
stream per GPU; at N GPUs each rank runs its own stream (independent streams,
no collective on the frame path; "scaling": "weak").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

value  : aggregate panorama frames/s with the input frames resident in HBM
         (device-to-device path, stitch_b200_process_device), CUDA-event timed
         on the context stream, max over ranks.
e2e    : the same metric through the reference-facing C-ABI call
         (stitch_b200_process) with pinned HOST frames: H2D of every camera
         frame + D2H of the balanced panorama (RGB + mask) inside the timed
         region, max over ranks.
--impl reference : the CPU oracle (the reference's path restated in C; the
         reference itself needs Eigen3 and cannot be built here) on the box's
         host cores, same workload, rank 0 only.
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
    # BASELINE.json configs[3]
    "c4": dict(views=8, width=3840, height=2160, focal_scale=1.03,
               desc="8 cameras 3840x2160 RGB single panorama stream"),
}


def build_scene(wl, seed):
    import paper_2308_09209_b200 as pb

    spec = pb.SynthSpec(seed=seed, views=wl["views"], frames=300, width=wl["width"],
                        height=wl["height"], overlap_fraction=0.3,
                        perturb_focal_scale=wl["focal_scale"])
    spec.color_casts = [(1.0, 1.0, 1.0) if v % 2 == 0 else (0.88, 1.0, 1.08)
                        for v in range(wl["views"])]
    spec.flicker = [pb.FlickerEvent(frame=5, view=wl["views"] - 1, gains=(1.15, 1.1, 0.95))]
    spec.object = pb.ParallaxObject(enabled=True, half_size=0.08 * wl["width"] * 500 / (
        0.9 * wl["width"]), velocity=(4.0, 1.0))
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
def kernel_model(state, wl):
    """Algorithmic HBM bytes (and FP32 flops for the flow) per frame, per
    kernel family."""
    pairs = state.pairs
    o = [(p.bounds[2] - p.bounds[0]) * (p.bounds[3] - p.bounds[1]) for p in pairs]
    P = state.canvas_width * state.canvas_height
    inputs = wl["views"] * wl["width"] * wl["height"] * 3
    # flow pyramid pixel counts per task (2 directions per pair)
    lv_px = []
    for p in pairs:
        w, h = p.bounds[2] - p.bounds[0], p.bounds[3] - p.bounds[1]
        if w < 16 or h < 16:
            continue
        levels = [(w, h)]
        for _ in range(1, 4):
            if levels[-1][0] < 16 or levels[-1][1] < 16:
                break
            levels.append((max(1, levels[-1][0] // 2), max(1, levels[-1][1] // 2)))
        lv_px.append(sum(a * b for a, b in levels))
    flow_px = 2 * sum(lv_px)  # both directions
    sweeps = 10
    model = {
        # reads 3 B of source per warped pixel (both sides of each crop), writes uchar4
        "crop_warp": dict(bytes=sum(2 * (3 + 4) * n for n in o)),
        # reads two uchar4 crops
        "pair_stats": dict(bytes=sum(8 * n for n in o)),
        # reads raw crops, writes corrected crops + luma
        "flow_prepare": dict(bytes=sum(2 * (4 + 4 + 4) * n for n in o)),
        # per warp iteration: read u,v,a,b; write u,v (24 B/px); 5 iterations per level
        "hs_iter": dict(bytes=5 * 24 * flow_px,
                        flops=5 * flow_px * (sweeps * 18 + 40)),
        # inputs once, pano uchar4 write, overlap crops + flows + weights
        "canvas": dict(bytes=inputs + 4 * P + sum((8 + 16 + 4) * n for n in o)),
        # uchar4 pano read, RGB + mask write
        "tone": dict(bytes=8 * P),
    }
    return model


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
    from paper_2308_09209_b200 import _abi

    lib = _abi.load()
    torch.cuda.set_device(local_rank)
    wl = WORKLOADS[args.config]
    sc = build_scene(wl, seed=1 + rank)
    cfg = sc.config()
    cfg.device = local_rank
    nv = wl["views"]
    F = args.frame_sets
    threads = max(1, cpu_cores() // max(1, world))
    frame_bytes = wl["width"] * wl["height"] * 3
    # pre-render F frame sets, stage them in pinned host memory and in HBM
    host_sets, dev_sets = [], []
    for t in range(F):
        hs, ds = [], []
        for v in range(nv):
            img = sc.render_view(v, t, threads).data
            hp = lib.stitch_b200_host_alloc(frame_bytes)
            C.memmove(hp, img.ctypes.data, frame_bytes)
            dp = lib.stitch_b200_device_alloc(local_rank, frame_bytes)
            pb.pipeline.check(lib.stitch_b200_memcpy_h2d(dp, hp, frame_bytes))
            hs.append(hp)
            ds.append(dp)
        host_sets.append((C.c_void_p * nv)(*hs))
        dev_sets.append((C.c_void_p * nv)(*ds))
    first = [pb.Frame(np.zeros((wl["height"], wl["width"], 3), np.uint8)) for _ in range(nv)]
    state = pb.initialize(cfg, first)
    h = state.handle
    P = state.canvas_width * state.canvas_height
    out_rgb = lib.stitch_b200_host_alloc(P * 3)
    out_mask = lib.stitch_b200_host_alloc(P)
    stream = torch.cuda.ExternalStream(lib.stitch_b200_stream(h), device=local_rank)
    launches = state.launches_per_frame()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local_rank}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    clocks = ClockSampler(local_rank)
    clocks.start()
    # ---- warm-up ----
    for i in range(args.warmup):
        pb.pipeline.check(lib.stitch_b200_process_device(h, dev_sets[i % F], None))
    pb.pipeline.check(lib.stitch_b200_synchronize(h))
    # ---- timed: device-resident inputs ----
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    clocks.active = True
    e0.record(stream)
    for i in range(args.steps):
        pb.pipeline.check(lib.stitch_b200_process_device(h, dev_sets[i % F], None))
    e1.record(stream)
    torch.cuda.synchronize()
    clocks.active = False
    barrier()
    elapsed_ms = e0.elapsed_time(e1)
    max_ms = max_over_ranks(elapsed_ms)
    ms_per_step = max_ms / args.steps
    value = world * args.steps / (max_ms / 1e3)

    # ---- per-step latency distribution (p50) ----
    lat = []
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(min(args.steps, 200))]
    for i, (a, b) in enumerate(evs):
        a.record(stream)
        pb.pipeline.check(lib.stitch_b200_process_device(h, dev_sets[i % F], None))
        b.record(stream)
    torch.cuda.synchronize()
    lat = [a.elapsed_time(b) for a, b in evs]
    p50 = statistics.median(lat)

    # ---- e2e: reference-facing C-ABI call with pinned host buffers ----
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    for i in range(min(args.warmup, 3)):
        pb.pipeline.check(lib.stitch_b200_process(h, host_sets[i % F], out_rgb, out_mask, None))
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        pb.pipeline.check(lib.stitch_b200_process(h, host_sets[i % F], out_rgb, out_mask, None))
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    e2e_value = world * e2e_steps / e2e_s

    # ---- per-kernel profile (eager, CUDA events around each launch) ----
    n_ops = 4096
    kinds = (C.c_int * n_ops)()
    ms = (C.c_float * n_ops)()
    per_kind = {}
    prof_frames = 5
    for i in range(prof_frames):
        n = lib.stitch_b200_profile_frame(h, dev_sets[i % F], n_ops, kinds, ms)
        if n < 0:
            pb.pipeline.check(-n)
        for j in range(min(n, n_ops)):
            name = _abi.OP_KIND_NAMES[kinds[j]]
            d = per_kind.setdefault(name, [0.0, 0])
            d[0] += ms[j] / prof_frames
            d[1] += 1 if i == 0 else 0
    clocks.stop()

    peak, peak_kind = load_peaks()
    model = kernel_model(state, wl)
    total_kernel_ms = sum(v[0] for v in per_kind.values())
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
            k["fp32_gflops"] = round(mdl["flops"] / (t_ms * 1e-3) / 1e9, 1)
        kernels[name] = k
    dominant = max(per_kind, key=lambda n: per_kind[n][0])
    dk = kernels[dominant]
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(dominant)
    except Exception:
        pass
    roofline = {"kernel": dominant, "bound": "hbm",
                "achieved": dk.get("hbm_gbs"), "peak": peak, "unit": "GB/s",
                "frac": dk.get("hbm_frac"), "traffic": traffic,
                "peak_source": peak_kind,
                "alg_bytes_per_launch": (model[dominant]["bytes"] / max(1, dk["launches_per_frame"])
                                         if dominant in model else None)}
    hbm_kernels = {n: kernels[n] for n in ("canvas", "tone", "crop_warp", "pair_stats")
                   if n in kernels}

    result = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "p50_ms_per_frame": round(p50, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8 (fp64 warp, fp32 flow)",
        "data": "synthetic (procedural plane scene, SynthScene restatement; seeds 1..N)",
        "config": {"workload": wl["desc"], "config_key": args.config, "cameras": nv,
                   "camera_size": [wl["width"], wl["height"]],
                   "canvas": [state.canvas_width, state.canvas_height],
                   "pairs": [list(p.bounds) for p in state.pairs],
                   "streams_per_gpu": 1, "parallelism": f"stream-sharded x{world}",
                   "l2": (f"inputs cycle over {F} pre-rendered frame sets "
                          f"({F * nv * frame_bytes / 1e6:.0f} MB > 126 MB L2)")},
        "e2e": {"value": round(e2e_value, 2), "unit": UNIT,
                "h2d_bytes_per_step": nv * frame_bytes, "d2h_bytes_per_step": P * 4,
                "steps": e2e_steps},
        "gpu_launches": launches * args.steps,
        "kernels_per_frame": launches,
        "roofline": roofline,
        "hbm_kernels": hbm_kernels,
        "kernels": kernels,
        "clocks": clocks.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(args, wl, sample_seconds=args.cpu_seconds)
    return result


# ---------------------------------------------------------------------------
# CPU oracle (reference path restated in C) -- baseline only
# ---------------------------------------------------------------------------
def oracle_state_for(sc, threads):
    import oracle as O

    c = sc.config_c()
    cams = [(c.cams[v].fx, c.cams[v].fy, c.cams[v].cx, c.cams[v].cy, list(c.cams[v].rotation),
             list(c.cams[v].translation)) for v in range(c.n_views)]
    sizes = [(c.width[v], c.height[v]) for v in range(c.n_views)]
    return O.OracleState(O.make_config(c.n_views, c.reference, sizes, cams, threads=threads))


def cpu_baseline(args, wl, sample_seconds=15.0, max_frames=None):
    sc = build_scene(wl, seed=1)
    threads = cpu_cores()
    st = oracle_state_for(sc, threads)
    frames = [[sc.render_view(v, t, threads).data for v in range(wl["views"])]
              for t in range(2)]
    st.process(frames[0])  # warm-up (allocator, page faults)
    n, t0 = 0, time.perf_counter()
    while True:
        st.process(frames[n % 2])
        n += 1
        el = time.perf_counter() - t0
        if el >= sample_seconds or (max_frames and n >= max_frames):
            break
    st.close()
    return {"value": round(n / el, 4), "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{n} frames of the same workload after 1 warm-up frame "
                      f"({el:.1f} s, oracle/liboracle.so, {threads} OpenMP threads)"}


def run_reference(args):
    wl = WORKLOADS[args.config]
    sc = build_scene(wl, seed=1)
    threads = cpu_cores()
    st = oracle_state_for(sc, threads)
    frames = [[sc.render_view(v, t, threads).data for v in range(wl["views"])]
              for t in range(args.frame_sets if args.frame_sets < 4 else 4)]
    budget = args.ref_budget_s
    t_w = time.perf_counter()
    for i in range(args.warmup):
        st.process(frames[i % len(frames)])
        if time.perf_counter() - t_w > budget / 4:
            break
    n, t0 = 0, time.perf_counter()
    for i in range(args.steps):
        st.process(frames[i % len(frames)])
        n += 1
        if time.perf_counter() - t0 > budget:
            break
    el = time.perf_counter() - t0
    st.close()
    v = n / el
    return {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": UNIT,
            "n_gpus": 0, "steps": n, "warmup": args.warmup, "ms_per_step": round(1e3 * el / n, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8 (fp64 warp, fp32 flow)", "data": "synthetic",
            "config": {"workload": wl["desc"], "config_key": args.config},
            "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": threads,
                             "kind": "port",
                             "sample": f"{n} of {args.steps} requested frames within a "
                                       f"{budget:.0f} s budget (oracle/liboracle.so: the "
                                       "reference path restated in C; the reference needs "
                                       "Eigen3 and cannot be built here)"},
            "e2e": {"value": round(v, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--frame-sets", type=int, default=16)
    ap.add_argument("--e2e-steps", type=int, default=200)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-budget-s", type=float, default=120.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank != 0:
            return
        print(json.dumps(run_reference(args)))
        return
    if world > 1:
        import torch

        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl")
    res = run_b200(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(res))
    if world > 1:
        import torch

        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
