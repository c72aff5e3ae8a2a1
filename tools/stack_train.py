"""Deep-stack TRAINING step of the MUG-V 10B architecture on one B200 at BASELINE configs[3]'s 480p/2s shape
(latent 7 x 60 x 104 x 24 -> 10,920 tokens): the full FlowTrainer::step (flowtrain.cpp:231-282: forward through
`depth` blocks, backward, grad norm, AdamW) at tensor-parallel size 1, bf16, device-resident inputs.

The 56-block stack needs 319 GB at TP size 1 (mgv_plan_rank_bytes); depth 24 (~138 GB) is the deepest slice that
leaves headroom on one 180 GB B200, and every block does identical work, so ms/block here times 56 is the full
stack's single-GPU cost.  The per-rank plan at TP 2/4/8 (186 / 120 / 87 GB) is printed alongside.  Also checks the
context's own allocations (mgv_ctx_memory) against the planner for this depth.  Prints one JSON line.

    python tools/stack_train.py [--depth 24] [--steps 5] [--warmup 3] [--grid 16 45 80 --recompute]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--depth", type=int, default=24)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--grid", type=int, nargs=3, default=[7, 30, 52], help="token grid; 16 45 80 = 720p/5s (57,600)")
    ap.add_argument("--recompute", action="store_true", help="per-block activation recompute (mgv_ctx_set_recompute)")
    args = ap.parse_args()
    import numpy as np
    import torch
    from bench import ADAMW, TEXT_D, TEXT_L, ClockSampler
    from paper_2510_17519_b200.capi import (Context, make_flow_sample, mgv_flow_sample, paper_config,
                                             plan_rank_bytes, rng_uniform)
    from tools.stack_common import shared_stack_params

    grid = tuple(args.grid)
    N = grid[0] * grid[1] * grid[2]
    cfg = paper_config(depth=args.depth)
    H, D = cfg.hidden, cfg.patch_dim
    params = shared_stack_params(args.depth)
    ctx = Context(0, "bf16")
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    ctx.set_adamw(**ADAMW)
    ctx.set_recompute(args.recompute)
    ctx.upload(cfg, params)
    del params
    latent = rng_uniform(3, (grid[0], 2 * grid[1], 2 * grid[2], D // 4), -1.0, 1.0)
    rows, coords = ctx.latent_rows(latent)
    noise, t_val, _ = make_flow_sample(5, N, D)
    text = make_flow_sample(4, TEXT_L, TEXT_D)[0]
    d_clean = torch.tensor(rows, dtype=torch.float64, device="cuda")
    d_noise = torch.tensor(noise, dtype=torch.float64, device="cuda")
    d_text = torch.tensor(text, dtype=torch.float64, device="cuda")
    d_coords = torch.tensor(np.ascontiguousarray(coords, dtype=np.int32), device="cuda")
    ds = (mgv_flow_sample * 1)()
    for i in range(3):
        ds[0].dims[i] = grid[i]
    ds[0].coords, ds[0].clean_rows, ds[0].noise, ds[0].t = d_coords.data_ptr(), d_clean.data_ptr(), d_noise.data_ptr(), t_val
    torch.cuda.synchronize()
    step = lambda: ctx.flow_step_device(ds, d_text.data_ptr(), TEXT_L, 8.0)  # noqa: E731
    losses = []
    for _ in range(args.warmup):
        losses.append(step()[0])
    torch.cuda.synchronize()
    ctx.prof_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            loss, gn = step()
            losses.append(loss)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    prof = ctx.prof_stats()
    mem = ctx.memory()
    free, total = torch.cuda.mem_get_info(0)
    plan = plan_rank_bytes(cfg, "bf16", 1, N, TEXT_L, recompute=args.recompute)
    ctx.close()
    # algorithmic training FLOPs: 3x the forward's per block (28 N H^2 + 4 N^2 H + cross-attention)
    L = TEXT_L
    per_block_fwd = 28.0 * N * H * H + 4.0 * N * N * H + 4.0 * N * L * H + 2.0 * L * TEXT_D * 2 * H
    flops = 3.0 * args.depth * per_block_fwd
    out = {"what": f"FlowTrainer::step (fwd + bwd + grad norm + AdamW), {args.depth}-block slice of the 10B stack "
                   f"(H3456, 24x144 heads, FFN 13824, text 64x4096), {N} tokens (grid {grid}), bf16, TP size 1, 1 GPU, "
                   + ("per-block activation recompute (the extra block forwards are not counted in the FLOPs), "
                      if args.recompute else "") + "device-resident inputs, CUDA events",
           "depth": args.depth, "tokens": N, "recompute": bool(args.recompute), "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": ms, "ms_per_block": ms / args.depth, "tokens_per_s": N / (ms / 1e3),
           "tflops_algorithmic": flops / (ms / 1e3) / 1e12,
           "full_56_block_step_ms_projected": 56.0 * ms / args.depth,
           "loss_first_last": [losses[0], losses[-1]], "finite": bool(all(math.isfinite(x) for x in losses)),
           "grad_norm_last": gn,
           "memory_gb": {k: v / 1e9 for k, v in mem.items()},
           "plan_gb": {k: v / 1e9 for k, v in plan.items()},
           "device_used_gb": (total - free) / 1e9,
           "plan_56_per_rank_gb": {str(p): sum(plan_rank_bytes(paper_config(56), "bf16", p, N, L,
                                                               recompute=args.recompute).values()) / 1e9
                                   for p in (1, 2, 4, 8)},
           "phases_ms_per_step": {k: v["ms"] / args.steps for k, v in prof.items()},
           "clocks": clk.summary()}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    tag = f"stack_train_d{args.depth}_n{N}" + ("_rc" if args.recompute else "")
    with open(os.path.join(ROOT, "gpurun_out", f"{tag}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
