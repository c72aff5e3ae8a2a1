"""Tensor-parallel exchange on one B200 with emulated ranks (mgv_ctx_set_tp(P, 0, NULL)): the full flow step
(fwd + bwd + grad norm + AdamW) of the 10B-shaped block at 57,600 tokens, bf16, with the peer-memory exchange
(tp_peer.h) against the in-place accumulation of the partials (MGV_TP_EXCHANGE=nccl, which with emulated ranks
accumulates in the GEMM epilogue).  Reports ms per step and the exchange phase (signal + reduce/gather + wait
kernels) with its HBM rate: per exchange each of the P emulated owners reads P slots of ceil(N/P) x H fp32, and
the summed rows are written once (one result region when the ranks are emulated).  On a real TP group one
rank's owner reads N x H fp32 locally and writes N x H, (P-1)/P of it over NVLink.

    python tools/tp_exchange.py [--sizes 2 8] [--steps 3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", type=int, nargs="+", default=[2, 8])
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    import numpy as np
    import torch
    from bench import GRID, PATCH, TEXT_D, TEXT_L, grid_coords
    from paper_2510_17519_b200.capi import Context, mgv_flow_sample, paper_config

    cfg = paper_config(depth=1)
    gs = 0.2 * (12.0 / cfg.hidden) ** 0.5  # SURVEY 8(d) weights: init_dit_params(Rng(1)) + gates from Rng(2)
    U, Hp, Wp = GRID
    N, H = U * Hp * Wp, cfg.hidden
    rng = np.random.default_rng(100)
    d_clean = torch.tensor(rng.uniform(-1.0, 1.0, (N, PATCH)), dtype=torch.float64, device="cuda")
    d_noise = torch.tensor(rng.standard_normal((N, PATCH)), dtype=torch.float64, device="cuda")
    d_text = torch.tensor(np.random.default_rng(4).standard_normal((TEXT_L, TEXT_D)), dtype=torch.float64, device="cuda")
    d_coords = torch.tensor(grid_coords(GRID), device="cuda")
    ds = (mgv_flow_sample * 1)()
    for i in range(3):
        ds[0].dims[i] = GRID[i]
    ds[0].coords, ds[0].clean_rows, ds[0].noise, ds[0].t = d_coords.data_ptr(), d_clean.data_ptr(), d_noise.data_ptr(), 0.5
    out = {"workload": f"flow step, 10B block depth 1, {N} tokens, bf16, emulated TP ranks on one GPU", "runs": []}
    for P in args.sizes:
        for mode in ["nccl", "peer"]:
            os.environ["MGV_TP_EXCHANGE"] = mode
            ctx = Context(0, "bf16")
            stream = torch.cuda.Stream()
            ctx.set_stream(stream.cuda_stream)
            ctx.set_tp(P)
            ctx.init_params(cfg, seed=1, gate_seed=2, gate_std=gs, gate_b_std=gs / 4)
            step = lambda: ctx.flow_step_device(ds, d_text.data_ptr(), TEXT_L, 8.0)  # noqa: E731
            step()
            torch.cuda.synchronize()
            ctx.prof_enable(True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                loss, gn = step()
            e1.record(stream)
            torch.cuda.synchronize()
            prof = ctx.prof_stats()
            ctx.prof_enable(False)
            r = {"tp": P, "exchange": "peer" if mode == "peer" else "accumulate (emulated NCCL mode)",
                 "ms_per_step": e0.elapsed_time(e1) / args.steps, "loss": loss, "grad_norm": gn}
            if "tp_exchange" in prof:
                x = prof["tp_exchange"]
                rpr = -(-N // P)
                per = x["ms"] / x["launches"]
                if os.environ.get("MGV_TP_PAYLOAD") == "bf16":  # bf16 slots / result + the local widening pass
                    nbytes = (P * P * rpr * H + N * H) * 2 + N * H * (2 + 4)
                    r["payload"] = "bf16"
                else:
                    nbytes = (P * P * rpr * H + N * H) * 4  # P emulated owners each read P slots; one result write
                r["exchange_ms_per_call"] = per
                r["exchange_calls_per_step"] = x["launches"] / args.steps
                r["exchange_bytes_per_call"] = nbytes
                r["exchange_hbm_gbs"] = nbytes / (per * 1e-3) / 1e9
            out["runs"].append(r)
            print(json.dumps(r), flush=True)
            ctx.close()
            del ctx
            torch.cuda.empty_cache()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "tp_exchange.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
