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
args = ap.parse_args()
grid = tuple(int(x) for x in args.grid.split(","))
cfg = paper_config(depth=1)
ctx = Context(0, "bf16")
ctx.upload(cfg, bench.synthetic_params(cfg, 1234))
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
