#!/usr/bin/env python
"""Benchmark: DiT-block video tokens/s at the 57.6K-token 10B shape (BASELINE.json).

Workload (BASELINE.json configs[2]): one MUG-V-10B-shaped DiT block (H=3456,
24 heads x 144, FFN 13824, text 64 x 4096; depth 1 plus the patch / final /
velocity heads) on a 720p/5s latent 16x90x160x24 -> 16x45x80 = 57,600 tokens,
the full flow-matching training step: forward + backward + grad norm + AdamW
update (FlowTrainer::step, flowtrain.cpp:257-289, optim.cpp:7-24), one sample per GPU,
synthetic latents and random-init weights.  Multi-GPU = data parallel over
NCCL (weak scaling: one sample per rank; gradients all-reduced in-library).

  value : device-resident inputs (mgv_flow_step_device), CUDA events, max over ranks
  e2e   : the C-ABI call with pinned HOST buffers (mgv_flow_step): H2D of the
          sample + text and D2H of loss/grad-norm inside the timed region
  --impl reference : the unmodified reference (oracle/_ref, compiled from the
          reference sources) on the host cores, one process per core.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Under torchrun every rank runs; rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import ctypes
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
sys.path.insert(0, ROOT)

METRIC = "DiT-block video tokens/sec at 57.6K-token 10B shape; attention TFLOP/s vs peak"
GRID_720P = (16, 45, 80)  # token grid (U, H', W') of the 720p/5s latent (16, 90, 160, 24)
GRID = GRID_720P
H, HEADS, HD, TEXT_L, TEXT_D, PATCH = 3456, 24, 144, 64, 4096, 96
# AdamW hyper-parameters of the timed training step (optim.hpp:14-18 defaults, small lr)
ADAMW = dict(lr=1e-4, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0)
REF_SAMPLE = (2, 2, 4)  # bounded CPU sample: latent (U, h, w) = (2, 2, 4) x 24 ch -> grid 2x1x2 = 4 tokens


def peaks():
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            m = json.load(f)
        p.update({k: m[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in m})
        p["source"] = "measured"
    return p


# ------------------------------------------------------------------ distributed plumbing
def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        cmd = ["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
               "--format=csv,noheader,nounits"]
        while not self._stop.is_set():
            try:
                out = subprocess.run(cmd, capture_output=True, text=True, timeout=5).stdout.strip()
                sm, smax, reasons = [x.strip() for x in out.split(",")]
                self.samples.append((float(sm), float(smax), int(reasons, 16)))
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        mask = 0
        for s in self.samples:
            mask |= s[2]
        reasons = [v for k, v in self.REASONS.items() if mask & k and v != "gpu_idle"]
        return {"sm_mhz": statistics.median(s[0] for s in self.samples), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------ synthetic model + inputs
def grid_coords(dims):
    U, Hp, Wp = dims
    t, y, x = np.meshgrid(np.arange(U), np.arange(Hp), np.arange(Wp), indexing="ij")
    return np.stack([t.ravel(), y.ravel(), x.ravel()], 1).astype(np.int32)


def pinned(shape, dtype):
    import torch
    t = torch.empty(shape, dtype={np.float64: torch.float64, np.int32: torch.int32}[dtype], pin_memory=True)
    return t.numpy(), t


# ------------------------------------------------------------------ CPU baseline (oracle/_ref)
def _ref_worker(args):
    """One process = one reference model pinned to one host core (taskset -c <core>); times `steps` samples of
    REF_SAMPLE fwd+bwd+AdamW.  The reference library is loaded only in these child processes."""
    seed, steps, conn = args
    try:
        os.sched_setaffinity(0, {seed % (os.cpu_count() or 1)})
    except (AttributeError, OSError):
        pass
    from oracle import oracle as O
    if O.ref_lib() is None:
        conn.send("unavailable")
        conn.close()
        return
    cfg = O.paper_config(depth=1)
    gs = O.gate_std_for(cfg.hidden)
    ref = O.RefModel(cfg, 1 + seed, 2, gs, gs / 4)
    opt = O.RefAdamW(ADAMW["lr"], ADAMW["beta1"], ADAMW["beta2"], ADAMW["eps"], ADAMW["weight_decay"])
    text = O.Rng(4).normal_tensor((TEXT_L, TEXT_D))
    U, h, w = REF_SAMPLE
    g = O.Rng(3 + seed).uniform_tensor((U, h, w, 24), -1.0, 1.0)
    s = O.make_batch([g], 0.0, O.Rng(5 + seed))
    conn.send("ready")
    times = []
    for _ in range(steps):
        if conn.recv() != "go":
            break
        t0 = time.perf_counter()
        out = ref.flow_fwdbwd(s, text, 8.0, grads=True, with_V=False)
        opt.update_model(ref, out["grads"])  # the full FlowTrainer::step (flowtrain.cpp:257-282)
        times.append(time.perf_counter() - t0)
        conn.send(times[-1])
    conn.close()


def ref_tokens():
    U, h, w = REF_SAMPLE
    return U * (h // 2) * (w // 2)


def host_info():
    info = {"nproc": os.cpu_count()}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
        info["ram_gb"] = round(int(open("/proc/meminfo").read().split("MemTotal:")[1].split()[0]) / 1e6, 1)
    except Exception:
        pass
    return info


def _sweep_fit():
    """The committed single-core sweep of the reference (tools/cpu_sweep.py on a B200 host, profiles/): fitted
    t = a N + b N^2 and its extrapolations, labelled as such."""
    path = os.path.join(ROOT, "profiles", "cpu_sweep_r02.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        sw = json.load(f)
    return {k: sw[k] for k in ("fit", "extrapolated", "host", "source") if k in sw}


def cpu_baseline_once():
    """The reference (oracle/_ref, compiled from its unmodified sources) on ONE pinned host core, on the bounded
    sample; the reference is loaded only in the spawned child.  Falls back to the numpy port when the compiled
    reference is absent."""
    import multiprocessing as mp
    if os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libmugv_ref.so")):
        ctx = mp.get_context("spawn")
        a, b = ctx.Pipe()
        p = ctx.Process(target=_ref_worker, args=((0, 1, b),))
        p.start()
        if a.recv() == "ready":
            a.send("go")
            dt = a.recv()
            p.join()
            return {"value": ref_tokens() / dt, "unit": "tokens/s", "cores": 1, "kind": "reference",
                    "sample": f"reference FlowTrainer::step (fwd+bwd+AdamW), 10B dims depth 1, {ref_tokens()} tokens "
                              f"(latent {REF_SAMPLE[0]}x{REF_SAMPLE[1]}x{REF_SAMPLE[2]}x24), text 64x4096, "
                              f"1 thread pinned to core 0: {dt:.1f} s",
                    "host": host_info(), "sweep": _sweep_fit()}
        p.join()
    # numpy port (oracle.py) in a child when the compiled reference is absent
    ctx = mp.get_context("spawn")
    with ctx.Pool(1) as pool:
        dt = pool.apply(_port_sample)
    return {"value": ref_tokens() / dt, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"numpy fp64 port fwd+bwd, 10B dims depth 1, {ref_tokens()} tokens: {dt:.1f} s",
            "host": host_info()}


def _port_sample():
    from oracle import oracle as O
    cfg = O.paper_config(depth=1)
    P = O.open_gates(O.init_dit_params(cfg, O.Rng(1)), 2, O.gate_std_for(cfg.hidden), O.gate_std_for(cfg.hidden) / 4)
    g = O.Rng(3).uniform_tensor((REF_SAMPLE[0], REF_SAMPLE[1], REF_SAMPLE[2], 24), -1.0, 1.0)
    s = O.make_batch([g], 0.0, O.Rng(5))
    text = O.Rng(4).normal_tensor((TEXT_L, TEXT_D))
    t0 = time.perf_counter()
    O.flow_fwdbwd(P, cfg, s, text, 8.0, grads=True)
    return time.perf_counter() - t0


def run_reference(args, rank, world):
    if rank != 0:
        return
    import multiprocessing as mp
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libmugv_ref.so")):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libmugv_ref.so not built"}))
        return
    try:
        avail_gb = int(open("/proc/meminfo").read().split("MemAvailable:")[1].split()[0]) / 1e6
    except Exception:
        avail_gb = 64.0
    # per process: fp64 params 1.6 GB + grads 1.6 GB (+ a copy) + AdamW m, v 3.2 GB + activations
    procs_n = max(1, min(os.cpu_count() or 1, int(avail_gb // 24), 96))
    ctx = mp.get_context("spawn")
    steps = args.warmup + args.steps
    pipes, procs = [], []
    for i in range(procs_n):
        a, b = ctx.Pipe()
        p = ctx.Process(target=_ref_worker, args=((i, steps, b),))
        p.start()
        pipes.append(a)
        procs.append(p)
    def recv_all(timeout):
        for a, p in zip(pipes, procs):
            if not a.poll(timeout) or not p.is_alive() and not a.poll(0):
                raise RuntimeError(f"reference worker {p.pid} died or stalled (exit {p.exitcode})")
            a.recv()

    try:
        recv_all(600)
        step_s = []
        for k in range(steps):
            t0 = time.perf_counter()
            for a in pipes:
                a.send("go")
            recv_all(600)
            if k >= args.warmup:
                step_s.append(time.perf_counter() - t0)
    except (RuntimeError, EOFError, OSError) as e:
        for p in procs:
            p.kill()
        print(json.dumps({"impl": "reference", "unavailable": f"reference host run failed: {e}"}))
        return
    for p in procs:
        p.join()
    ms = 1000.0 * sum(step_s) / len(step_s)
    value = procs_n * ref_tokens() / (ms / 1000.0)
    sample = (f"{procs_n} processes x 1 reference sample each (FlowTrainer::step fwd+bwd+AdamW, 10B dims "
              f"depth 1, {ref_tokens()} tokens, text 64x4096) per step; bounded stand-in for the 57.6K-token sample, "
              f"which the reference cannot run (637 GB fp64 attention probabilities)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "10B DiT block training step: fwd+bwd+AdamW (reference CPU path, bounded sample)",
                   "tokens_per_sample": ref_tokens(), "parallelism": f"{procs_n} host processes"},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": procs_n, "kind": "reference", "sample": sample,
                         "host": host_info(), "sweep": _sweep_fit()},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


# ------------------------------------------------------------------ our arm
def rank_groups(rank, world, tp):
    """rank = dp_rank * tp + tp_rank: a TP group is tp consecutive ranks (one node's NVLink peers), DP joins the
    ranks holding the same tp_rank.  Returns (tp_rank, dp_rank, dp_world, tp_root, dp_root); the roots are the
    global ranks (tp_rank 0 of this TP group, dp_rank 0 of this DP group) whose NCCL ids the group uses."""
    if tp < 1 or world % tp:
        raise ValueError(f"--tp {tp} does not divide the {world} ranks")
    tp_rank, dp_rank = rank % tp, rank // tp
    return tp_rank, dp_rank, world // tp, dp_rank * tp, tp_rank


def run_ours(args, rank, world, local):
    import torch
    from paper_2510_17519_b200.capi import (Context, FlowSample, make_flow_sample, mgv_flow_sample, paper_config,
                                             rng_uniform)

    def rng_normal_text():  # Rng(4).normal_tensor({64, 4096}) == make_batch noise draws of Rng(4) (no t / mask use)
        return make_flow_sample(4, TEXT_L, TEXT_D)[0]

    torch.cuda.set_device(local)
    GRID = tuple(args.grid)
    tp = args.tp
    # rank = dp_rank * tp + tp_rank: a TP group is tp consecutive ranks; DP joins the ranks with the same tp_rank
    try:
        tp_rank, dp_rank, dp_world, tp_root, dp_root = rank_groups(rank, world, tp)
    except ValueError as e:
        sys.exit(f"bench.py: {e}")
    cfg = paper_config(depth=args.depth)
    ctx = Context(local, "bf16")
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    if world > 1:
        import torch.distributed as dist
        ids = [None] * world
        # rank r offers the TP id of its group (if tp_rank == 0) and the DP id of its DP group (if dp_rank == 0)
        mine = (Context.nccl_unique_id() if tp > 1 and tp_rank == 0 else None,
                Context.nccl_unique_id() if dp_world > 1 and dp_rank == 0 else None)
        dist.all_gather_object(ids, mine)
        if tp > 1:
            ctx.set_tp(tp, tp_rank, ids[tp_root][0])
        if dp_world > 1:
            ctx.set_dp(dp_rank, dp_world, ids[dp_root][1])
    ctx.set_adamw(**ADAMW)  # the timed step is the full FlowTrainer::step: fwd + bwd + grad norm + AdamW
    if args.recompute:
        ctx.set_recompute(True)
    # SURVEY 8(d) weights: init_dit_params(cfg, Rng(1)) + gates opened from Rng(2) at the width-scaled std
    gs = 0.2 * math.sqrt(12.0 / cfg.hidden)
    ctx.init_params(cfg, seed=1, gate_seed=2, gate_std=gs, gate_b_std=gs / 4)

    U, Hp, Wp = GRID
    N = U * Hp * Wp
    # SURVEY 8(d) inputs with the reference's Rng streams: latent Rng(3 + rank).uniform_tensor(16x90x160x24, -1, 1)
    # patchified on device (dit::latent_rows), text Rng(4).normal_tensor (64 x 4096), noise and t from
    # make_batch(Rng(5 + rank)) (flowtrain.cpp:231-250); rank r > 0 draws its own sample
    latent = rng_uniform(3 + dp_rank, (U, 2 * Hp, 2 * Wp, PATCH // 4), -1.0, 1.0)
    rows, coords = ctx.latent_rows(latent)
    noise, t_val, _ = make_flow_sample(5 + dp_rank, N, PATCH)
    clean_h, clean_t = pinned((N, PATCH), np.float64)
    noise_h, noise_t = pinned((N, PATCH), np.float64)
    text_h, text_t = pinned((TEXT_L, TEXT_D), np.float64)
    coords_h, coords_t = pinned((N, 3), np.int32)
    clean_h[:] = rows
    noise_h[:] = noise
    text_h[:] = rng_normal_text()
    coords_h[:] = coords
    # device-resident copies for the `value` figure
    d_clean, d_noise = clean_t.cuda(), noise_t.cuda()
    d_text, d_coords = text_t.cuda(), coords_t.cuda()
    ds = (mgv_flow_sample * 1)()
    for i in range(3):
        ds[0].dims[i] = GRID[i]
    ds[0].coords, ds[0].clean_rows, ds[0].noise, ds[0].t = d_coords.data_ptr(), d_clean.data_ptr(), d_noise.data_ptr(), t_val
    torch.cuda.synchronize()

    def step_dev():
        return ctx.flow_step_device(ds, d_text.data_ptr(), TEXT_L, 8.0)

    for _ in range(args.warmup):
        step_dev()
    barrier(world)
    torch.cuda.synchronize()
    ctx.prof_enable(True)
    launches = 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            loss, gnorm = step_dev()
            launches += ctx.last_step_launches()
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps, world)
    prof = ctx.prof_stats()
    ctx.prof_enable(False)
    value = dp_world * N / (ms / 1000.0)

    # e2e through the public C ABI with pinned host buffers
    sample = FlowSample(GRID, coords_h, clean_h, noise_h, t_val, None)
    for _ in range(min(args.warmup, 2)):
        ctx.flow_step([sample], text_h, 8.0)
    barrier(world)
    e2e_s = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        out = ctx.flow_step([sample], text_h, 8.0)
        e2e_s.append(time.perf_counter() - t0)
    e2e_ms = max_over_ranks(1000.0 * sum(e2e_s) / len(e2e_s), world)
    h2d = clean_h.nbytes + noise_h.nbytes + coords_h.nbytes + text_h.nbytes
    d2h = 16  # loss + grad norm

    if rank != 0:
        return
    pk = peaks()
    kern = {}
    for name, st in prof.items():
        per = st["ms"] / max(1, st["launches"])
        kern[name] = {"ms_per_step": st["ms"] / args.steps, "ms_per_launch": per, "share": st["ms"] / args.steps / ms}
    # algorithmic FLOPs per launch: self-attention fwd 4 N^2 H, bwd 8 N^2 H (a TP rank: its H / tp)
    f_fwd, f_bwd = 4.0 * N * N * H / tp, 8.0 * N * N * H / tp
    att = {}
    if "attn_fwd" in kern:
        att["fwd_tflops"] = f_fwd / (kern["attn_fwd"]["ms_per_launch"] * 1e9)
    if "attn_bwd" in kern:
        att["bwd_tflops"] = f_bwd / (kern["attn_bwd"]["ms_per_launch"] * 1e9)
    if "gemm" in prof and "attn_fwd" in prof and "attn_bwd" in prof:
        # the north star's "attention + MLP" figure: self-attention fwd + bwd (algorithmic) and every bf16 GEMM
        # (2 M N K: all linears fwd, dgrad, wgrad) over the device time of exactly those launches
        g = prof["gemm"]
        t_ms = (g["ms"] + prof["attn_fwd"]["ms"] + prof["attn_bwd"]["ms"]) / args.steps
        fl = (g["flops"] + f_fwd * prof["attn_fwd"]["launches"] + f_bwd * prof["attn_bwd"]["launches"]) / args.steps
        att["tensor_kernels"] = {"tflops": fl / (t_ms * 1e9), "frac": fl / (t_ms * 1e9) / pk["bf16_tflops_sustained"],
                                 "ms_per_step": t_ms, "share_of_step": t_ms / ms,
                                 "gemm_tflops": g["flops"] / (g["ms"] * 1e9), "gemm_launches_per_step": g["launches"] / args.steps,
                                 "what": "self-attention fwd+bwd + all bf16 GEMMs, algorithmic FLOPs / their device time"}
    cands = {k: v for k, v in kern.items() if k in ("attn_fwd", "attn_bwd")}
    dom = max(cands, key=lambda k: cands[k]["ms_per_step"]) if cands else None
    roof = None
    if dom:
        fl = f_fwd if dom == "attn_fwd" else f_bwd
        achieved = fl / (kern[dom]["ms_per_launch"] * 1e9)
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "kernel_traffic.json")
        if os.path.exists(tpath):
            traffic = json.load(open(tpath)).get(dom)
        roof = {"kernel": dom, "bound": "tensor", "achieved": achieved, "peak": pk["bf16_tflops_sustained"],
                "unit": "TFLOP/s", "frac": achieved / pk["bf16_tflops_sustained"], "traffic": traffic,
                "peak_source": f"{pk['source']} bf16_tflops_sustained (kernel timed inside a long step)",
                "flops_per_launch": fl}
    total_flops = 3 * (28.0 * N * H * H + 4.0 * N * N * H + 4.0 * N * TEXT_L * H + 2 * TEXT_L * TEXT_D * 2 * H)
    total_flops *= args.depth / tp
    par = f"dp{dp_world}" if tp == 1 else f"tp{tp}" + (f"xdp{dp_world}" if dp_world > 1 else "")
    shape = {(16, 45, 80): "720p/5s latent 16x90x160x24 -> 57600 tokens",
             (7, 30, 52): "480p/2s latent 7x60x104x24 -> 10920 tokens"}.get(GRID, f"token grid {GRID} -> {N} tokens")
    stack = "depth 1" if args.depth == 1 else f"{args.depth}-block stack"
    res = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic latents + random-init 10B-shaped weights",
        "config": {"workload": f"MUG-V 10B DiT block (H3456, 24x144 heads, FFN 13824, text 64x4096), {stack} + "
                               f"patch/final/velocity heads, {shape}, flow-matching "
                               "fwd+bwd + grad norm + AdamW update (the full FlowTrainer::step), 1 sample per "
                               + ("GPU" if tp == 1 else f"TP group of {tp}"),
                   "tokens_per_sample": N, "samples_per_gpu": 1 if tp == 1 else 1.0 / tp, "global_batch": dp_world,
                   "parallelism": par, "depth": args.depth, "recompute": bool(args.recompute),
                   "l2": "working set ~17 GB >> 126 MB L2 (no flush needed)"},
        "roofline": roof,
        "attention": att,
        "block_tflops": total_flops / (ms * 1e9),
        "kernels": kern,
        "cpu_baseline": None,
        "e2e": {"value": dp_world * N / (e2e_ms / 1000.0), "unit": "tokens/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "clocks": clk.summary(),
        "gpu_launches": launches,
        "loss": loss, "grad_norm": gnorm,
    }
    if world == 1 and args.depth == 1 and GRID == GRID_720P and not args.no_extra:
        res["extra_configs"] = extra_configs(ctx, args)
    if world == 1 and not args.no_cpu_baseline:
        try:
            res["cpu_baseline"] = cpu_baseline_once()
        except Exception as e:  # the baseline is reported, never required
            res["cpu_baseline"] = {"value": None, "unavailable": str(e)[:200]}
    print(json.dumps(res))


def extra_configs(ctx, args):
    """BASELINE.json configs[1] (480p/2s forward, 10,920 tokens) and configs[4] (mixed-resolution varlen
    batch with first-frame conditioning) through the public C ABI with host buffers (e2e timing)."""
    import torch
    from paper_2510_17519_b200.capi import FlowSample
    out = {}
    rng = np.random.default_rng(7)
    text = np.random.default_rng(4).standard_normal((TEXT_L, TEXT_D))
    # configs[1]: predict_velocity (forward only) on a 480p/2s latent (7, 60, 104, 24) -> 7x30x52 = 10920 tokens
    dims = (7, 30, 52)
    n = dims[0] * dims[1] * dims[2]
    rows = rng.uniform(-1, 1, (n, PATCH))
    coords = grid_coords(dims)
    tau = np.full(n, 0.5)
    for _ in range(2):
        ctx.predict_velocity(rows, coords, dims, text, tau, 8.0)
    ts = []
    for _ in range(max(3, args.steps)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.predict_velocity(rows, coords, dims, text, tau, 8.0)
        ts.append(time.perf_counter() - t0)
    ms = 1000 * statistics.median(ts)
    f_fwd = 28.0 * n * H * H + 4.0 * n * n * H + 4.0 * n * TEXT_L * H
    out["cfg1_480p_fwd"] = {"workload": "predict_velocity, 10B dims depth 1, latent 7x60x104x24 -> 10920 tokens",
                            "tokens_per_s": n / (ms / 1000), "ms": ms, "block_tflops": f_fwd / (ms * 1e9),
                            "timing": "wall clock around the C-ABI call, host buffers (e2e)"}
    # configs[4]: mixed-resolution batch: 4 x 480p/2s clips + 4 x 720p images, first-frame mask prob 0.3
    shapes = [(7, 30, 52)] * 4 + [(1, 45, 80)] * 4
    samples = []
    for k, d in enumerate(shapes):
        nn = d[0] * d[1] * d[2]
        co = grid_coords(d)
        cond = (co[:, 0] == 0).astype(np.uint8) if (d[0] > 1 and rng.uniform() < 0.3) else None
        samples.append(FlowSample(d, co, rng.uniform(-1, 1, (nn, PATCH)), rng.standard_normal((nn, PATCH)),
                                  float(rng.uniform(0.05, 0.95)), cond))
    tot = sum(s.clean_rows.shape[0] for s in samples)
    for packed in (True, False):
        ctx.set_varlen(packed)
        ctx.flow_step(samples, text, 8.0)
        ts = []
        for _ in range(max(3, args.steps)):
            t0 = time.perf_counter()
            ctx.flow_step(samples, text, 8.0)
            ts.append(time.perf_counter() - t0)
        ms = 1000 * statistics.median(ts)
        key = "cfg4_varlen_mixed" if packed else "cfg4_sequential"
        how = ("ONE packed step: 256-row-aligned segments, block-diagonal attention (mgv_ctx_set_varlen)" if packed
               else "samples run one after another (varlen off)")
        out[key] = {"workload": "flow step fwd+bwd over 4 x (7,30,52) clips + 4 x (1,45,80) images "
                                f"= {tot} tokens, first-frame conditioning p=0.3, {how}",
                    "tokens_per_s": tot / (ms / 1000), "ms": ms,
                    "timing": "wall clock around the C-ABI call, host buffers (e2e)"}
    ctx.set_varlen(False)
    return out


def _relaunch_under_torchrun(args):
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-exec as N ranks over NCCL on this node (the driver's
    own launch line) and return its exit code."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the configs[1]/configs[4] side measurements")
    ap.add_argument("--tp", type=int, default=1, help="tensor-parallel group size (head/column TP over NCCL + NVLink "
                                                      "peer exchange); the other factor of --gpus is DP")
    ap.add_argument("--depth", type=int, default=1, help="DiT blocks (configs[3]: 56, with --grid 7 30 52)")
    ap.add_argument("--recompute", action="store_true", help="per-block activation recompute (deep stacks at 57.6K)")
    ap.add_argument("--grid", type=int, nargs=3, default=list(GRID_720P), metavar=("U", "H", "W"),
                    help="token grid (latent / 2x2 patches); 7 30 52 = the 480p/2s shape")
    args = ap.parse_args()
    if args.gpus < 1:
        sys.exit("bench.py: --gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        if args.impl == "ours":
            import torch
            if torch.cuda.device_count() < args.gpus:
                sys.exit(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, {torch.cuda.device_count()} visible")
        sys.exit(_relaunch_under_torchrun(args))
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if world_env != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but the launcher started {world_env} ranks")
    if args.impl == "ours":
        import torch
        if torch.cuda.device_count() < world_env:
            sys.exit(f"bench.py: {world_env} ranks need {world_env} GPUs, {torch.cuda.device_count()} visible")
    rank, world, local = dist_init()
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
