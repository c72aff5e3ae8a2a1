"""One warm-up + N profiled device-resident steps of the bench workload (for ncu launch lists)."""
import argparse
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_17519_b200.capi import Context, mgv_flow_sample, paper_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--grid", default="16,45,80")
ap.add_argument("--kernels", action="store_true")
ap.add_argument("--fusions", type=int, default=None, help="mgv_dev_set_fusions mask (A/B of the forward fusions)")
args = ap.parse_args()
if args.fusions is not None:
    from paper_2510_17519_b200._lib import lib
    lib().mgv_dev_set_fusions(args.fusions)
grid = tuple(int(x) for x in args.grid.split(","))
cfg = paper_config(depth=1)
ctx = Context(0, "bf16")
gs = 0.2 * (12.0 / cfg.hidden) ** 0.5
ctx.init_params(cfg, seed=1, gate_seed=2, gate_std=gs, gate_b_std=gs / 4)
N = grid[0] * grid[1] * grid[2]
rng = np.random.default_rng(0)
d_clean = torch.tensor(rng.uniform(-1, 1, (N, 96)), device="cuda")
d_noise = torch.tensor(rng.standard_normal((N, 96)), device="cuda")
d_text = torch.tensor(rng.standard_normal((64, 4096)), device="cuda")
d_coords = torch.tensor(bench.grid_coords(grid), device="cuda")
ds = (mgv_flow_sample * 1)()
for i in range(3):
    ds[0].dims[i] = grid[i]
ds[0].coords, ds[0].clean_rows, ds[0].noise, ds[0].t = d_coords.data_ptr(), d_clean.data_ptr(), d_noise.data_ptr(), 0.5
for k in range(1 + args.steps):
    loss, gn = ctx.flow_step_device(ds, d_text.data_ptr(), 64, 8.0)
    print(f"step {k}: loss {loss:.6f} grad_norm {gn:.6f} ms {ctx.last_step_ms():.2f} launches {ctx.last_step_launches()}")

if args.kernels and args.steps > 0:
    # per-kernel device time over `steps` profiled steps (CUPTI activity records)
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for k in range(args.steps):
            ctx.flow_step_device(ds, d_text.data_ptr(), 64, 8.0)
        torch.cuda.synchronize()
    tot, cnt = {}, {}
    per = __import__("os").environ.get("PER_LAUNCH")
    for e in prof.events():
        if per and e.device_type.name == "CUDA" and per in e.name:
            print(f"  launch {e.device_time_total / 1000.0:9.3f} ms  {e.name[:60]}")
        if e.device_type.name == "CUDA":
            tot[e.name] = tot.get(e.name, 0.0) + e.device_time_total / 1000.0
            cnt[e.name] = cnt.get(e.name, 0) + 1
    T = sum(tot.values())
    print(f"total kernel time per step: {T / args.steps:.2f} ms")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:int(__import__("os").environ.get("TOPK", "40"))]:
        print(f"  {v / args.steps:8.3f} ms {100 * v / T:5.1f}% x{cnt[k] // args.steps:3d}  {k[:110]}")
