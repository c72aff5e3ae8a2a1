"""Full-depth MUG-V 10B stack (56 blocks, dit.cpp:40-48) on one B200: predict_velocity (dit.hpp:104-106)
through the C ABI at the 480p/2s (10,920 tokens) and 720p/5s (57,600 tokens) shapes -- BASELINE configs[3] at
tensor-parallel size 1 (forward only: training all 56 blocks needs the TP split).

Weights: one block of init_dit_params + opened gates (tools/stack_common.py) shared by all 56 block names on the host, so host
memory stays ~2 GB while the device holds 56 independent fp32 masters + bf16 copies (+ the fp32 gradient
buffer the context allocates), ~110 GB.  Timing: wall clock around the C-ABI call with host fp64 buffers
(the e2e figure), after one warm-up call.  Prints one JSON line.
Usage: python tools/stack_fwd.py [reps]"""
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2510_17519_b200.capi import Context, paper_config  # noqa: E402
from tools.stack_common import shared_stack_params  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
DEPTH = 56
cfg = paper_config(depth=DEPTH)
params = shared_stack_params(DEPTH)
n_params = sum(v.size for k, v in params.items())

import torch  # noqa: E402

ctx = Context(0, "bf16")
t0 = time.perf_counter()
ctx.upload(cfg, params)
upload_s = time.perf_counter() - t0
free, total = torch.cuda.mem_get_info(0)
H, L, TD = cfg.hidden, 64, cfg.text_dim
text = np.random.default_rng(4).standard_normal((L, TD))
out = {"what": "predict_velocity, full 56-block 10B stack (H3456, 24x144 heads, FFN 13824, text 64x4096), bf16, "
               "1 GPU (TP size 1), host fp64 buffers, wall clock around the C-ABI call",
       "params": int(n_params), "upload_s": upload_s, "device_mem_used_gb": (total - free) / 1e9, "shapes": {}}
for name, grid in [("480p_2s", (7, 30, 52)), ("720p_5s", (16, 45, 80))]:  # token grids after 2x2 patchify
    U, Hp, Wp = grid
    N = U * Hp * Wp
    rng = np.random.default_rng(3)
    rows = rng.uniform(-1.0, 1.0, (N, cfg.patch_dim))
    coords = bench.grid_coords(grid)
    ts = np.full(N, 0.5)
    v = ctx.predict_velocity(rows, coords, grid, text, ts)  # warm-up (workspace sizing)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        v = ctx.predict_velocity(rows, coords, grid, text, ts)
        times.append(time.perf_counter() - t0)
    s = min(times)
    # algorithmic forward FLOPs: per block 28 N H^2 + 4 N^2 H + cross-attention; heads + gmlp/mod ~ 0
    per_block = 28.0 * N * H * H + 4.0 * N * N * H + 4.0 * N * L * H + 2.0 * L * TD * 2 * H
    flops = DEPTH * per_block + 2.0 * N * H * H + 4.0 * N * cfg.patch_dim * H
    out["shapes"][name] = {"tokens": N, "s_per_call": s, "all_s": times, "tokens_per_s": N / s,
                           "tflops": flops / s / 1e12, "finite": bool(np.isfinite(v).all()),
                           "v_rms": float(math.sqrt(float((v * v).mean())))}
ctx.close()
print(json.dumps(out))
