#!/usr/bin/env python
"""Benchmark of the S3R-GS streamlined per-view splatting path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config av2] [--impl s3r|reference]

One step = one s3r_render_batch of this rank's views of the config's scene:
temporal filter -> instance projection + LOD + life update -> depth sort ->
supertile binning -> alpha blend (every row of SURVEY.md §8(a)).  Inputs are
resident in HBM before the timed region (scene 168 MB at C3, larger than the
126 MB L2; each step also writes ~4 GB of images), so no L2 flush is needed
between steps (smaller scenes are flushed).

Multi-GPU (BASELINE configs C3/C4): the configured global batch (C3 64 views,
C4 256, C2 100) is split into contiguous shards of the (frame, camera)-sorted
views, one per rank (strong scaling, the default; --scaling weak keeps
--views per rank instead).  Gaussians are replicated; views are independent,
so there is no data-path collective.  `python bench.py --gpus N` without a
torchrun environment re-launches itself under torch.distributed.run with N
ranks (S3R_DIST_BACKEND=gloo runs the ranks on fewer GPUs as a functional
test); under torchrun WORLD_SIZE must equal --gpus.  Rank 0 prints one JSON
line.

--impl reference times the CPU oracle (oracle/, single-threaded C) on host
cores: one view of the same workload per step.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2503_08217_b200 import scenegen as sg  # noqa: E402

METRIC = "rendered views/sec and Gaussians/sec at 1/2/4/8 B200; % HBM/FP32 roofline"
UNIT = "views/s"
# FP32 operations per blend evaluation for the roofline: SURVEY.md §8(d)'s
# algorithmic count for Eq.2 with an exact exponential, ~28 per E_alg (FMA = 2):
# dx, dy 2; power 5; clamp 1; exp 10; alpha clamp 1; w 1; colour + depth 6;
# T 1; termination 1.  The R-ARITH step as the kernel executes it costs 36
# (exp2 polynomial 14 instead of 10, the o 2^n multiply, the exp2 scaling)
# and is reported beside it (EXEC_FLOPS_PER_EVAL) but is not the roofline's.
FLOPS_PER_EVAL = 28
EXEC_FLOPS_PER_EVAL = 36
# ... and of its adjoint (k_raster_bwd): dy, e2 6; clamp 1; exp2 14; o G 1;
# alpha 1; 1 - alpha 1; rcp 1; T_before 1; w 1; c.gC 6; rest 2; dL/dalpha 2;
# R 2; colour sums 6; opacity 2; power 1; dy moments 5; flush test 1.
BWD_FLOPS_PER_EVAL = 54
SM_COUNT_B200 = 148
GLOBAL = {"views": 0}        # views of one step over all ranks (set in main)


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled through NVML every
    50 ms during the timed region (the same counters nvidia-smi reports)."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.stop_ev = threading.Event()
        self.err = None

    def start(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = self.index
            if vis:
                ids = [x for x in vis.split(",") if x.strip()]
                if idx < len(ids) and ids[idx].strip().isdigit():
                    idx = int(ids[idx])
            self.h = N.nvmlDeviceGetHandleByIndex(idx)
            self.smax = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception as e:           # noqa: BLE001
            self.err = f"nvml unavailable: {e}"
            return
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        N = self.N
        bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap,
                "hw_power_brake_slowdown": N.nvmlClocksEventReasonHwPowerBrakeSlowdown}
        while not self.stop_ev.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
                util = N.nvmlDeviceGetUtilizationRates(self.h).gpu
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, util))
                for k, b in bits.items():
                    if r & b:
                        self.reasons.add(k)
            except Exception as e:       # noqa: BLE001
                self.err = str(e)
                break
            time.sleep(0.05)

    def stop(self):
        if self.err and not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.err}
        self.stop_ev.set()
        self.t.join(timeout=2)
        sm = [s for s, _ in self.samples]
        loaded = [s for s, u in self.samples if u > 50] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": float(self.smax), "reasons": sorted(self.reasons),
                "samples": len(sm), "source": "NVML, 50 ms period"}


def stage_bytes(stats, views, n_scene, n_distinct_t, pair_passes):
    # depth sort passes over (depth bits << gbits | index): 32 + bits(N) key bits
    depth_passes = math.ceil((32 + max(1, (max(n_scene, 2) - 1).bit_length())) / 8)
    """Algorithmic bytes per stage for one batch (DESIGN.md §Roofline)."""
    Nt = sum(s["n_temporal"] for s in stats)
    Nv = sum(s["n_visible"] for s in stats)
    Nr = sum(s["n_rendered"] for s in stats)
    Ps = sum(s["n_bin_pairs"] for s in stats)
    P = sum(s["n_pairs"] for s in stats)
    px = sum(v.width * v.height for v in views)
    tiles = sum(((v.width + 15) // 16) * ((v.height + 15) // 16) for v in views)
    # K1 writes each distinct time's list once
    nt_distinct = sum({v.t: s["n_temporal"] for v, s in zip(views, stats)}.values())
    return {
        "filter": 8 * n_scene * math.ceil(max(n_distinct_t, 1) / 64) + 4 * nt_distinct,
        "project": 56 * Nt + 8 * Nv + (16 + 48 + 8) * Nr,
        "depth_sort": 8 * Nr + depth_passes * 24 * Nr,
        # permute (order + record in/out + rectangle) + count + scatter (rect + 4 B per
        # supertile pair) + expand (supertile list + rectangle in, 4 B per tile pair out)
        "bin": (4 + 48 + 48 + 8) * Nr + 8 * Nr + 8 * Nr + 4 * Ps + 12 * Ps + 4 * P,
        # tile lists (4 B per pair), unique records, images
        "raster": 4 * P + 48 * Nr + 20 * px,
        # NeurF query (when on): own-frame mean + id in, colour float4 out
        "color": 32 * Nr,
    }


def run_reference(args, rank):
    """The oracle as it stands, on host cores, one view per step."""
    if rank != 0:
        return
    import oracle
    cfg_name = args.config
    scene, views = sg.make_config(cfg_name, n_views=max(args.views, 1))
    W = args.warmup
    K = args.steps
    for i in range(W):
        oracle.render_view(scene, views[i % len(views)], "f32", pairs=False)
    t0 = time.perf_counter()
    for i in range(K):
        oracle.render_view(scene, views[(W + i) % len(views)], "f32", pairs=False)
    dt = time.perf_counter() - t0
    v = K / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": K, "warmup": W, "ms_per_step": 1e3 * dt / K, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg_name, "n_gaussians": scene.n,
                   "image": f"{views[0].width}x{views[0].height}", "views_per_step": 1},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"1 view of {cfg_name} per step, single-threaded C oracle"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_conventional(args, ctx, ds, views, outs, world, dev, stream, streamlined_value):
    """NEXT-2: the same views through the conventional pipeline (per-view world
    transform of every dynamic Gaussian, all Gaussians projected, no temporal
    filter, no LOD) — the paper's baseline (Fig.1a); `speedup` is the
    streamlined views/s over this one (the paper's central claim, Fig.4)."""
    import torch
    import torch.distributed as dist
    from paper_2503_08217_b200 import s3r
    tabs = list(s3r.conventional_tables(views, device=dev))
    ctx.set_pipeline(True)
    try:
        for _ in range(2):
            ctx.render_batch(ds, views, tabs, outs)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        k = max(2, min(args.steps, 5))
        ctx.set_timing(True)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(k)]
        for a, b in evs:
            a.record(stream)
            ctx.render_batch(ds, views, tabs, outs)
            b.record(stream)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in evs)
        st = ctx.stage_times()
        ctx.set_timing(False)
        ctx.set_counters(True)
        ctx.render_batch(ds, views, tabs, outs)
        torch.cuda.synchronize()
        stats = [ctx.stats(i) for i in range(len(views))]
        ctx.set_counters(False)
    finally:
        ctx.set_pipeline(False)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = GLOBAL["views"] * k / (ms / 1e3)
    renders = max(st["renders"], 1)
    return {"metric": "conventional-pipeline views/s (world transform + project all, no "
                      "temporal filter, no LOD)", "value": value, "unit": UNIT,
            "ms_per_step": ms / k, "steps": k, "speedup": streamlined_value / value,
            "stages_ms": {s_: st[s_] / renders for s_ in s3r.STAGES},
            "workload_per_view": {q: sum(s[q] for s in stats) / len(views) for q in
                                  ("n_temporal", "n_visible", "n_rendered", "n_pairs",
                                   "n_blend_evals")}}


def random_neurf_params(num_instances, dev, seed=11):
    """Random weights of the R22 NeurF shapes (no trained weights here), made
    on the device; He-style scales keep activations O(1)."""
    import torch
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    r = lambda *sh, s=1.0: torch.randn(*sh, generator=g, device=dev) * s
    p = {"w1": r(2, 64, 64, s=(2 / 44) ** 0.5), "b1": r(2, 64, s=0.1),
         "w2": r(2, 64, 64, s=(2 / 64) ** 0.5), "b2": r(2, 64, s=0.1),
         "w3": r(2, 3, 64, s=(2 / 64) ** 0.5), "b3": r(2, 3, s=0.1),
         "time_emb": r(16, 8), "class_emb": r(num_instances, 4)}
    p["w1"][:, :, 43:] = 0
    p["pos_scale"] = 100.0
    return p


def run_neurf(args, ctx, ds, scene, views, tables, outs, world, dev, stream, peaks):
    """NEXT-4: the streamlined render with the NeurF colour query (k_neurf on
    the tcgen05 tensor cores, random weights of the R22 architecture)."""
    import torch
    import torch.distributed as dist
    prm = random_neurf_params(scene.num_instances, dev)
    ctx.set_neural_colors(prm)
    try:
        for _ in range(2):
            ctx.render_batch(ds, views, tables, outs)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        k = max(2, min(args.steps, 5))
        ctx.set_timing(True)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(k)]
        for a, b in evs:
            a.record(stream)
            ctx.render_batch(ds, views, tables, outs)
            b.record(stream)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in evs)
        st = ctx.stage_times()
        ctx.set_timing(False)
        stats = [ctx.stats(i) for i in range(len(views))]
    finally:
        ctx.set_neural_colors(None)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    renders = max(st["renders"], 1)
    color_ms = st["color"] / renders
    rows = sum(s["n_rendered"] for s in stats)
    tiles = sum((s["n_rendered"] + 127) // 128 for s in stats)
    # executed: both networks on every 128-row tile (N = 128, 128, 32; K = 64)
    exec_flops = tiles * 128 * 2 * 64 * (128 + 128 + 32)
    alg_flops = rows * 2 * (64 * 64 + 64 * 64 + 64 * 3)      # one network per Gaussian
    peak = float(peaks.get("bf16_tflops", 1695.8))
    return {"metric": "views/s with the NeurF colour query (tcgen05 bf16 MLP, NEXT-4)",
            "value": GLOBAL["views"] * k / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / k,
            "color_stage_ms": color_ms, "rows_per_step": rows,
            "roofline": {"kernel": "k_neurf", "bound": "tensor",
                         "achieved": exec_flops / (color_ms / 1e3) / 1e12 if color_ms else None,
                         "peak": peak, "unit": "TFLOP/s",
                         "frac": exec_flops / (color_ms / 1e3) / 1e12 / peak if color_ms else None,
                         "peak_source": "MEASURED_PEAKS.json bf16_tflops (cuBLAS bf16 burst)",
                         "exec_flops_per_launch": exec_flops, "alg_flops_per_launch": alg_flops,
                         "alg_bytes_per_launch": 32 * rows}}


def run_fast_exp(args, ctx, ds, views, tables, outs, world, dev, stream, exact_value, E_alg):
    """The same render with the SFU exponential in K7 (s3r_set_fast_exp, DESIGN.md
    R24): not bit-exact with the oracle (images within 1e-4), reported beside
    the exact headline as SURVEY.md §8(c) asks."""
    import torch
    import torch.distributed as dist
    ctx.set_fast_exp(True)
    try:
        for _ in range(2):
            ctx.render_batch(ds, views, tables, outs)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        k = max(3, min(args.steps, 10))
        ctx.set_timing(True)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(k)]
        for a, b in evs:
            a.record(stream)
            ctx.render_batch(ds, views, tables, outs)
            b.record(stream)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in evs)
        st = ctx.stage_times()
        ctx.set_timing(False)
    finally:
        ctx.set_fast_exp(False)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = GLOBAL["views"] * k / (ms / 1e3)
    raster_ms = st["raster"] / max(st["renders"], 1)
    return {"metric": "views/s with the SFU exponential in the rasterizer (s3r_set_fast_exp)",
            "value": value, "unit": UNIT, "ms_per_step": ms / k, "steps": k,
            "raster_ms": raster_ms, "speedup_vs_exact": value / exact_value,
            "blend_evals_per_s": E_alg / (raster_ms / 1e3) if raster_ms else None,
            "parity": "RGB, final T within 1e-4 of the oracle; depth within 1e-4 x deepest splat "
                      "at termination flips; decisions / order / life bit-exact "
                      "(tests/test_gpu_parity.py::test_fast_exp_within_tolerance)"}


def load_traffic(kernel, workload):
    """DRAM bytes per launch of `kernel` from the committed ncu capture of this
    bench command (profiles/ncu_traffic.json, written by tools/ncu_traffic.py);
    None unless the capture ran the same workload."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            allk = json.load(f)
        # the exact-exp forward is k_raster<0,0,0> (k_raster<0,0> before the fast-exp mode)
        names = [kernel] if isinstance(kernel, str) else list(kernel)
        d = next(allk[n] for n in names if n in allk)
        if d.get("workload", "av2") != workload:
            return None, None
        return d["dram_bytes_per_launch"], d["source"]
    except (OSError, KeyError, ValueError, StopIteration):
        return None, None


def scene_instances(ds):
    return int(ds.num_instances)


def run_train(args, ctx, ds, views, tables, outs, world, dev, stream):
    from paper_2503_08217_b200 import parallel
    """Config 5: one step = training forward of the batch, MSE against noisy
    targets (s3r_mse), backward of blend + projection (s3r_render_backward)
    and, for N > 1, an NCCL all-reduce (SUM) of the per-Gaussian gradients."""
    import torch
    import torch.distributed as dist
    gen = torch.Generator(device=dev)
    gen.manual_seed(5)
    # the batch's images, targets and image gradients each live in one flat
    # buffer (per-view slices), so that the MSE is ONE s3r_mse call per step
    sizes = [v.height * v.width * 3 for v in views]
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    rgb_all = torch.empty(int(offs[-1]), device=dev)
    # (the loss is on RGB: the training render writes no depth / final-T images)
    outs = [{"rgb": rgb_all[offs[i]:offs[i + 1]].view(v.height, v.width, 3)}
            for i, v in enumerate(views)]
    ctx.render_batch(ds, views, tables, outs)
    targets_all = torch.clamp(rgb_all + 0.05 * torch.randn(rgb_all.shape, generator=gen,
                                                           device=dev), 0, 1)
    gimg_all = torch.empty_like(rgb_all)
    gimg = [gimg_all[offs[i]:offs[i + 1]].view(v.height, v.width, 3)
            for i, v in enumerate(views)]
    grads = {k: torch.zeros_like(getattr(ds, k)) for k in
             ("means_opacity", "scales", "rotations", "colors")}
    # NEXT-1 pose gradient: dL/d(instance camera table) per view and instance
    grads["table"] = torch.zeros((len(views), scene_instances(ds), 12), device=dev)
    loss = torch.zeros(1, device=dev)
    npix = sum(v.width * v.height * 3 for v in views)
    cots = [{"rgb": g} for g in gimg]
    ctx.set_training(True)
    e_fwd = [torch.cuda.Event(enable_timing=True) for _ in range(4)]

    def step():
        for g in grads.values():
            g.zero_()
        loss.zero_()
        e_fwd[0].record(stream)
        ctx.render_batch(ds, views, tables, outs)
        e_fwd[1].record(stream)
        ctx.mse(rgb_all, targets_all, 1.0 / npix, gimg_all, loss)
        e_fwd[2].record(stream)
        ctx.render_backward(ds, views, tables, cots, grads)
        e_fwd[3].record(stream)
        if world > 1:
            # per-Gaussian gradients are summed over ranks; the pose gradient is
            # per view (each rank owns its views' poses) and stays local
            parallel.allreduce_grads(grads)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms, fwd_ms, bwd_ms = 0.0, 0.0, 0.0
    for _ in range(args.train_steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        torch.cuda.synchronize()
        ms += a.elapsed_time(b)
        fwd_ms += e_fwd[0].elapsed_time(e_fwd[1])
        bwd_ms += e_fwd[2].elapsed_time(e_fwd[3])
    ctx.set_training(False)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    k = args.train_steps
    return {"metric": "training views/s (forward + MSE + backward"
                      + (f" + {dist.get_backend().upper()} grad all-reduce" if world > 1 else "")
                      + ")",
            "value": GLOBAL["views"] * k / (ms / 1e3), "unit": "views/s",
            "ms_per_step": ms / k, "forward_ms": fwd_ms / k, "backward_ms": bwd_ms / k,
            "loss": float(loss.item()), "views_per_gpu_per_step": len(views), "steps": k,
            "grads": "mean, opacity, scales, quaternion, colour (14 fp32 per Gaussian) + "
                     "instance-camera pose (12 fp32 per instance per view)"}


def _oracle_one(args):
    """One oracle render in a worker process (fork: the scene is inherited)."""
    import oracle
    i = args
    t = time.perf_counter()
    oracle.render_view(_CPU_SCENE, _CPU_VIEWS[i % len(_CPU_VIEWS)], "f32", pairs=False)
    return time.perf_counter() - t


_CPU_SCENE, _CPU_VIEWS = None, None


def cpu_baseline(cfg_name, procs=None):
    """The oracle as it stands on the host cores: P single-threaded renders of
    distinct views run concurrently in P forked processes (P = usable cores, at
    most 16; ~10-30 s); value = views / wall time."""
    import multiprocessing as mpr
    global _CPU_SCENE, _CPU_VIEWS
    _CPU_SCENE, _CPU_VIEWS = sg.make_config(cfg_name, n_views=16)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    P = max(1, min(procs or cores, 16))
    import oracle
    oracle.lib()                       # build / load once before forking
    t0 = time.perf_counter()
    with mpr.get_context("fork").Pool(P) as pool:
        per = pool.map(_oracle_one, range(P))
    dt = time.perf_counter() - t0
    v = _CPU_VIEWS[0]
    return {"value": P / dt, "unit": UNIT, "cores": P, "kind": "oracle",
            "per_view_single_core_s": sum(per) / len(per),
            "sample": f"{P} view(s) of {cfg_name} ({_CPU_SCENE.n} Gaussians, {v.width}x{v.height}), "
                      f"one single-threaded C oracle render per process, {P} processes, "
                      f"{dt:.1f} s wall"}


def view_shards(global_views: int, world: int, scaling: str, per_rank=None):
    """(offset, count) of every rank's views and the step's global view count.
    strong: the configured global batch in contiguous shards of the (frame,
    camera)-sorted views (same-t views co-locate; the first ranks take one
    more when it does not divide); weak: `per_rank` (default the global batch)
    views on every rank."""
    if scaling == "weak":
        per = per_rank if per_rank is not None else global_views
        return [(r * per, per) for r in range(world)], per * world
    base, extra = divmod(global_views, world)
    shards, off = [], 0
    for r in range(world):
        cnt = base + (1 if r < extra else 0)
        shards.append((off, cnt))
        off += cnt
    return shards, global_views


def relaunch(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: run this command again as N ranks
    under torch.distributed.run (one process per GPU, 127.0.0.1 rendezvous)."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="s3r", choices=["s3r", "reference"])
    ap.add_argument("--config", default="av2", choices=["toy", "street", "av2", "drive"])
    ap.add_argument("--views", type=int, default=None,
                    help="views per GPU per step (implies --scaling weak)")
    ap.add_argument("--scaling", default=None, choices=["strong", "weak"],
                    help="strong (default): the config's global batch split over the ranks")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--pool", type=int, default=4, help="distinct view batches cycled per step")
    ap.add_argument("--no-train", action="store_true", help="skip the config-5 training step")
    ap.add_argument("--no-neurf", action="store_true",
                    help="skip the NeurF colour-query measurement (NEXT-4)")
    ap.add_argument("--no-fast-exp", action="store_true",
                    help="skip the SFU-exponential variant (s3r_set_fast_exp)")
    ap.add_argument("--no-conventional", action="store_true",
                    help="skip the conventional-pipeline comparison (NEXT-2)")
    ap.add_argument("--train-steps", type=int, default=5)
    ap.add_argument("--mode", default="graph", choices=["graph", "sync"],
                    help="graph: capacity mode (s3r_set_capacity, sized from a warm-up batch "
                         "x 1.1) with each view batch captured once in a CUDA graph and "
                         "replayed; sync: the default synchronous sizing (two host readbacks "
                         "per batch)")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "s3r":
        sys.exit(relaunch(args.gpus))
    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        sys.exit(2)
    args.warmup = max(args.warmup, 3)
    if args.scaling is None:
        args.scaling = "weak" if args.views is not None else "strong"
    if args.impl == "reference":
        if args.views is None:
            args.views = 1
        run_reference(args, rank)
        return
    # global batch of the config (BASELINE: C3 64 views, C4 256, C2 all 100 frames)
    global_views = {"toy": 1, "street": sg.CONFIGS["street"].n_views, "av2": 64,
                    "drive": sg.CONFIGS["drive"].n_views}[args.config]
    shards, global_views = view_shards(global_views, world, args.scaling, args.views)
    args.views = shards[rank][1]
    GLOBAL["views"] = global_views
    if args.views < 1:
        print(f"bench.py: {global_views} views cannot be split over {world} ranks",
              file=sys.stderr)
        sys.exit(2)

    import torch
    import torch.distributed as dist
    from paper_2503_08217_b200 import s3r

    if os.environ.get("S3R_DIST_BACKEND") and torch.cuda.device_count():
        local = local % torch.cuda.device_count()    # functional multi-rank test on fewer GPUs
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("S3R_DIST_BACKEND", "nccl")   # gloo: functional test on one GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    # ---------------- workload (identical scene on every rank; views sharded)
    if args.config == "toy":
        scene, base_views = sg.make_toy()
        pools = [base_views * args.views]
    else:
        cfg = sg.CONFIGS[args.config]
        scene, traj = sg.make_street_scene(cfg)
        pools = []
        s0, sn = shards[rank]
        for p in range(args.pool):
            allv = sg.make_views(cfg, traj, n_views=global_views, seed=cfg.seed + 101 * p)
            pools.append(allv[s0:s0 + sn])
    ctx = s3r.Context(local)
    ds = s3r.DeviceScene.from_numpy(scene, device=dev)
    tables = [list(s3r.view_tables(ctx, vs, device=dev)) for vs in pools]
    outs = s3r.alloc_outputs(pools[0], device=dev)
    torch.cuda.synchronize()

    def step_eager(i):
        p = i % len(pools)
        ctx.render_batch(ds, pools[p], tables[p], outs)

    step = step_eager
    for i in range(args.warmup):
        step_eager(i)
    torch.cuda.synchronize()
    graphs = None
    if args.mode == "graph":
        # capacities: what every batch of the pool needed, x 1.1 (any overflow is
        # reported by s3r_check after the timed region and fails the run)
        need = None
        for p in range(len(pools)):
            step_eager(p)
            c_p = ctx.capacity_from_last(1.1)
            need = c_p if need is None else {k: max(need[k], c_p[k]) for k in need}
        ctx.set_capacity(need)
        graphs = []
        side = torch.cuda.Stream(device=dev)
        for p in range(len(pools)):
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                step_eager(p)                 # capacity-mode scratch + staging in place
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                step_eager(p)
            graphs.append(g)
        for g in graphs:
            g.replay()
        torch.cuda.synchronize()
        if ctx.check() != 0:
            raise RuntimeError("capacity mode overflowed during the warm-up")

        def step(i):
            graphs[i % len(graphs)].replay()
    capacity = ctx.capacity_from_last(1.0) if args.mode == "graph" else None
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    ctx.set_timing(True)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    # A scene smaller than L2 (toy, street) is flushed from L2 between timed
    # steps (a 256 MiB write, outside the per-step event pairs); the C3/C4 scenes
    # (168 MB / 840 MB) and the ~4 GB of images per step exceed the 126 MB L2.
    flush = scene.n * 84 < 126 * 2**20
    flush_buf = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device=dev) if flush else None
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    e0.record(stream)
    for i in range(args.steps):
        if flush:
            flush_buf.fill_(float(i))
        evs[i][0].record(stream)
        step(args.warmup + i)
        evs[i][1].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    stage_src = "CUDA events per stage inside the timed steps"
    if graphs is not None:
        # graph replays carry no per-stage events: the stage breakdown (and the
        # roofline's rasterizer time) comes from the same K steps rendered eagerly
        # in the capacity mode right after the timed region
        if ctx.check() != 0:
            raise RuntimeError("capacity mode overflowed during the timed steps")
        ctx.set_timing(True)
        for i in range(args.steps):
            if flush:
                flush_buf.fill_(float(i))
            step_eager(args.warmup + i)
        torch.cuda.synchronize()
        stage_src = ("CUDA events per stage of the same K steps rendered eagerly in the capacity "
                     "mode after the timed graph replays")
    st_times = ctx.stage_times()
    ctx.set_timing(False)
    ctx.set_capacity(None)
    rank_ms = {"max": ms / args.steps, "mean": ms / args.steps, "min": ms / args.steps}
    if world > 1:
        # load balance over ranks (front vs side cameras, near vs far content):
        # every rank's step time; `value` uses the max (the job's time)
        allt = [torch.zeros(1, device=dev, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allt, torch.tensor([ms], device=dev, dtype=torch.float64))
        per = [float(x.item()) / args.steps for x in allt]
        rank_ms = {"max": max(per), "mean": sum(per) / world, "min": min(per)}
        ms = max(per) * args.steps
        dist.barrier()
    views_per_step = len(pools[0])
    value = global_views * args.steps / (ms / 1e3)

    # ---------------- workload statistics + roofline (untimed render with counters)
    ctx.set_counters(True)
    ctx.render_batch(ds, pools[0], tables[0], outs)
    torch.cuda.synchronize()
    stats = [ctx.stats(i) for i in range(views_per_step)]
    ctx.set_counters(False)
    n_t = len({v.t for v in pools[0]})
    max_tiles = max(((v.width + 15) // 16) * ((v.height + 15) // 16) for v in pools[0])
    pair_passes = max(1, math.ceil(max(1, (max_tiles - 1).bit_length()) / 8))
    bytes_ = stage_bytes(stats, pools[0], scene.n, n_t, pair_passes)
    renders = max(st_times["renders"], 1)
    stage_ms = {k: st_times[k] / renders for k in s3r.STAGES}
    E_alg = sum(s["n_blend_evals"] for s in stats)
    E_exec = sum(s["n_blend_exec"] for s in stats)
    peaks, peak_src = load_peaks()
    sm_max = float(clocks.get("sm_max_mhz") or peaks.get("sm_max_mhz", 1965.0))
    alu_peak = SM_COUNT_B200 * 128 * 2 * sm_max * 1e6 / 1e12   # TFLOP/s
    hbm_peak = float(peaks["hbm_gbs"])
    stages = {}
    for k in s3r.STAGES:
        t_s = stage_ms[k] / 1e3
        stages[k] = {"ms": stage_ms[k], "alg_bytes": bytes_[k],
                     "GBps": bytes_[k] / t_s / 1e9 if t_s > 0 else None}
    stages["raster"]["TFLOPs"] = FLOPS_PER_EVAL * E_alg / (stage_ms["raster"] / 1e3) / 1e12 \
        if stage_ms["raster"] > 0 else None
    stages["raster"]["TFLOPs_executed_form"] = EXEC_FLOPS_PER_EVAL * E_alg / \
        (stage_ms["raster"] / 1e3) / 1e12 if stage_ms["raster"] > 0 else None
    dom = max(s3r.STAGES, key=lambda k: stage_ms[k])
    if dom == "raster":
        ach = stages["raster"]["TFLOPs"]
        roof = {"kernel": "k_raster", "bound": "alu", "achieved": ach, "peak": alu_peak,
                "unit": "TFLOP/s", "frac": ach / alu_peak,
                "peak_source": f"148 SMs x 128 FP32 lanes x 2 x {sm_max:.0f} MHz (B200_PROFILING.md unit counts)",
                "alg_flops_per_launch": FLOPS_PER_EVAL * E_alg, "traffic": None,
                "flops_per_eval": f"{FLOPS_PER_EVAL} (SURVEY.md §8(d), exact-exp Eq.2) x E_alg "
                                  f"{E_alg} per launch; the executed R-ARITH form is "
                                  f"{EXEC_FLOPS_PER_EVAL} (frac "
                                  f"{EXEC_FLOPS_PER_EVAL / FLOPS_PER_EVAL * ach / alu_peak:.3f})"}
        tr, tr_src = load_traffic(("k_raster<0,0,0,4>", "k_raster<0,0,0>", "k_raster<0,0>"),
                                  args.config)
        if tr is not None:
            roof["traffic"] = tr
            roof["traffic_source"] = f"{tr_src} (ncu --set full, one launch of this command)"
            roof["alg_bytes_per_launch"] = bytes_["raster"]
    else:
        ach = stages[dom]["GBps"]
        roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                "frac": ach / hbm_peak, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})",
                "alg_bytes_per_launch": bytes_[dom], "traffic": None}
        if args.config == "toy":
            roof["note"] = ("C1 (1,024 Gaussians, 16 tiles, one view per step) is latency-bound "
                            "in every kernel; the HBM fraction of its largest stage is not a "
                            "meaningful efficiency measure (DESIGN.md §10c)")

    # ---------------- config 5: training step (forward + MSE + backward [+ grad all-reduce])
    train = None
    if not args.no_train and args.config != "toy":
        train = run_train(args, ctx, ds, pools[0], tables[0], outs, world, dev, stream)
        # the backward rasterizer revisits the forward's evaluations (same E_alg)
        # back to front: FP32 roofline of the whole backward against them
        bw_s = train["backward_ms"] / 1e3
        train["roofline"] = {
            "kernel": "k_raster_bwd (+ k_project_bwd)", "bound": "alu",
            "achieved": BWD_FLOPS_PER_EVAL * E_alg / bw_s / 1e12, "peak": alu_peak,
            "unit": "TFLOP/s", "frac": BWD_FLOPS_PER_EVAL * E_alg / bw_s / 1e12 / alu_peak,
            "alg_flops_per_launch": BWD_FLOPS_PER_EVAL * E_alg,
            "note": f"{BWD_FLOPS_PER_EVAL} FLOP per evaluation (bench.py BWD_FLOPS_PER_EVAL)"}

    # ---------------- the SFU-exponential variant of the same render
    fast_exp = None
    if not args.no_fast_exp:
        fast_exp = run_fast_exp(args, ctx, ds, pools[0], tables[0], outs, world, dev, stream,
                                value, E_alg)

    # ---------------- NEXT-2: the conventional pipeline on the same views
    conventional = None
    if not args.no_conventional and args.config != "toy":
        conventional = run_conventional(args, ctx, ds, pools[0], outs, world, dev, stream, value)

    # ---------------- NEXT-4: NeurF colour query on the tensor cores
    neurf_line = None
    if not args.no_neurf and args.config != "toy":
        neurf_line = run_neurf(args, ctx, ds, scene, pools[0], tables[0], outs, world, dev, stream,
                               peaks)

    # ---------------- e2e through the host-buffer C-ABI entry point
    e2e = None
    if not args.no_e2e:
        hs = scene.copy()
        pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
        for k in ("means_opacity", "scales", "rotations", "colors", "instance_ids", "visibility",
                  "life"):
            setattr(hs, k, pin(np.ascontiguousarray(getattr(hs, k))))
        htabs = [[t.cpu().pin_memory().numpy() for t in tb] for tb in tables]
        hout = [{"rgb": torch.empty((v.height, v.width, 3), dtype=torch.float32,
                                    pin_memory=True).numpy()} for v in pools[0]]
        def estep(i):
            p = i % len(pools)
            ctx.render_batch_host(hs, pools[p], htabs[p], hout)
        for i in range(2):
            estep(i)
        if world > 1:
            dist.barrier()
        k_e2e = max(2, min(args.steps, 5))
        t0 = time.perf_counter()
        for i in range(k_e2e):
            estep(i)
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        h2d = sum(getattr(hs, k).nbytes for k in ("means_opacity", "scales", "rotations", "colors",
                                                   "instance_ids", "visibility", "life"))
        h2d += sum(t.nbytes for t in htabs[0])
        d2h = sum(o["rgb"].nbytes for o in hout) + hs.life.nbytes
        e2e = {"value": global_views * k_e2e / dt, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "steps": k_e2e, "api": "s3r_render_batch_host (pinned host buffers)"}

    # ---------------- end of a sweep (Eq.5 merge across ranks, Eq.6 commit): once per
    # pass over the trajectory, not per step, so timed separately (last: it
    # changes the scene's intervals)
    from paper_2503_08217_b200 import parallel
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    if world > 1:
        parallel.merge_life(ds.life, ctx.life_flip)
    ctx.commit_visibility(ds, 0.1)
    e1.record(stream)
    torch.cuda.synchronize()
    sweep_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([sweep_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sweep_ms = float(t.item())
    sweep_end = {"ms": sweep_ms, "ops": ("life merge: " + dist.get_backend().upper() +
                                         " all-reduce MAX over 2N floats + " if world > 1 else "")
                 + "commit (Eq.6, k_commit)", "allreduce_bytes": 8 * scene.n if world > 1 else 0}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.config != "toy":
        cpu = cpu_baseline(args.config)
    if rank == 0:
        n_scene = scene.n
        depth_passes = math.ceil((32 + max(1, (max(n_scene, 2) - 1).bit_length())) / 8)
        # views whose a4 runs in one CTA (k_small.cu): <= 2048 splats, <= 1024
        # tiles, splats x tiles <= 2^18 (s3r_internal.cuh small_view)
        def _small(st, v):
            nt = ((v.width + 15) // 16) * ((v.height + 15) // 16)
            return st["n_rendered"] <= 2048 and nt <= 1024 and st["n_rendered"] * nt <= (1 << 18)
        small = [_small(st, v) for st, v in zip(stats, pools[0])]
        any_small, all_small = any(small), all(small)
        # K1 (one launch of slot groups on a scene of < 296 filter tiles, else one
        # per 64 distinct times) + K2 + raster + the two plans / readbacks (one
        # plan when, in the capacity mode, every view plans itself in k_small) +
        # k_small + (hist, scan, depth passes, permute, count, scan, scatter,
        # expand) for the other views
        plans = 1 if (all_small and graphs is not None) else 2
        k1 = 1 if math.ceil(n_scene / 4096) < 296 else math.ceil(max(n_t, 1) / 64)
        launches_per_step = (k1 + 1 + 1 + plans
                             + (1 if any_small else 0)
                             + (0 if all_small else 2 + depth_passes + 5))
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.config, "n_gaussians": n_scene,
                       "instances": scene.num_instances - 1,
                       "image": f"{pools[0][0].width}x{pools[0][0].height}",
                       "views_per_gpu_per_step": views_per_step, "global_views_per_step":
                       global_views, "views_per_rank": [n for _, n in shards],
                       "parallelism": f"views sharded x{world}, Gaussians replicated",
                       "dist": ({"backend": dist.get_backend(), "ranks": dist.get_world_size()}
                                if world > 1 else None),
                       "l2": ("L2 flushed between timed steps (256 MiB write outside the "
                              "per-step CUDA-event pairs): scene smaller than L2") if flush else
                             f"inputs larger than L2 (scene {scene.n * 84 / 1e6:.0f} MB > 126 MB; "
                             "images written every step)"},
            "gaussians_per_s": n_scene * value,
            "processed_gaussians_per_s": sum(s["n_temporal"] for s in stats) / views_per_step * value,
            "clocks": clocks,
            "rank_ms_per_step": rank_ms,
            "gpu_launches": launches_per_step * args.steps,
            "mode": ("capacity mode + one CUDA graph per view batch (no host sync in a step; "
                     f"capacities {capacity})" if graphs is not None else
                     "synchronous sizing (two host readbacks per batch)"),
            "stage_times_source": stage_src,
            "roofline": roof,
            "stages": stages,
            "workload_per_view": {k: sum(s[k] for s in stats) / views_per_step for k in
                                  ("n_temporal", "n_visible", "n_lod_small", "n_lod_dropped",
                                   "n_rendered", "n_pairs", "n_bin_pairs", "n_blend_evals",
                                   "n_blend_exec")},
            "e2e": e2e,
            "cpu_baseline": cpu,
            "train": train,
            "conventional": conventional,
            "neurf": neurf_line,
            "fast_exp": fast_exp,
            "sweep_end": sweep_end,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
