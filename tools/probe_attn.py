"""Attention fwd/bwd probe at a given token count (default: the bench's 57,600), 24 heads x 144.
Usage: python tools/probe_attn.py [N] [fwd|bwd|both] [reps]"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_17519_b200._lib import lib  # noqa: E402

L = lib()
import os  # noqa: E402
P = ctypes.c_void_p
i64 = ctypes.c_int64
N = int(sys.argv[1]) if len(sys.argv) > 1 else 57600
what = sys.argv[2] if len(sys.argv) > 2 else "both"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
H, heads, hd = 3456, 24, 144
stream = torch.cuda.current_stream().cuda_stream
g = torch.Generator(device="cuda").manual_seed(0)
qkv = torch.randn(N, 3 * H, device="cuda", generator=g)
# unit-norm q/k per head with temperature ~ 10 (what the QK-norm produces) so the softmax is realistic
q = qkv[:, :2 * H].view(N, 2 * heads, hd)
q.div_(q.norm(dim=-1, keepdim=True))
q[:, :heads] *= 10.0
qkv = qkv.bfloat16()
o = torch.empty(N, H, device="cuda").bfloat16()
lse = torch.empty(heads, (N + 127) // 128 * 128, device="cuda")
lse_ld = lse.stride(0)


def timeit(fn, reps):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


fwd = lambda: L.mgv_dev_attn_fwd(1, P(qkv.data_ptr()), i64(3 * H), P(qkv[:, H:].data_ptr()), i64(3 * H),
                                 P(qkv[:, 2 * H:].data_ptr()), i64(3 * H), P(o.data_ptr()), i64(H),
                                 P(lse.data_ptr()), N, N, heads, hd, P(stream))
fwd()
if what in ("fwd", "both"):
    ms = timeit(fwd, reps)
    print(f"attn fwd N={N}: {ms:8.3f} ms  {4.0 * N * N * H / ms / 1e9:7.1f} TFLOP/s")
if what in ("bwd", "both"):
    dO = (torch.randn(N, H, device="cuda", generator=g) * 0.1).bfloat16()
    Dv = torch.empty(heads, (N + 127) // 128 * 128, device="cuda")
    dqkv = torch.empty(N, 3 * H, device="cuda").bfloat16()
    bwd = lambda: L.mgv_dev_attn_bwd(1, P(qkv.data_ptr()), i64(3 * H), P(qkv[:, H:].data_ptr()), i64(3 * H),
                                     P(qkv[:, 2 * H:].data_ptr()), i64(3 * H), P(o.data_ptr()), i64(H),
                                     P(lse.data_ptr()), P(dO.data_ptr()), i64(H), P(Dv.data_ptr()),
                                     P(dqkv.data_ptr()), i64(3 * H), P(dqkv[:, H:].data_ptr()), i64(3 * H),
                                     P(dqkv[:, 2 * H:].data_ptr()), i64(3 * H), P(0), 1, N, N, heads, hd, P(stream))
    ms = timeit(bwd, reps)
    print(f"attn bwd N={N}: {ms:8.3f} ms  {8.0 * N * N * H / ms / 1e9:7.1f} TFLOP/s (algorithmic 8N^2H)")

if len(sys.argv) > 4 and sys.argv[4] == "kernels":
    # per-kernel device time (CUPTI activity records), averaged over `reps` calls
    from torch.profiler import ProfilerActivity, profile
    fns = []
    if what in ("fwd", "both"):
        fns.append(fwd)
    if what in ("bwd", "both"):
        fns.append(bwd)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            for fn in fns:
                fn()
        torch.cuda.synchronize()
    tot = {}
    for e in prof.events():
        if e.device_type.name == "CUDA":
            tot[e.name] = tot.get(e.name, 0.0) + e.device_time_total / 1000.0
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]:
        print(f"  {v / reps:9.3f} ms  {k[:90]}")
