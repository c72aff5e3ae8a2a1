"""Kernel-level timing probe at the 10B block shape (N=57600, H=3456, 24x144): CUDA events, warm."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_17519_b200._lib import lib  # noqa: E402

L = lib()
P = ctypes.c_void_p
N, H, heads, hd = 57600, 3456, 24, 144
dev = "cuda"
stream = torch.cuda.current_stream().cuda_stream


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def gemm(A, a_mn, B, b_mn, M, Nn, K, C):
    return lambda: L.mgv_dev_gemm(1, P(A.data_ptr()), A.stride(0), a_mn, P(B.data_ptr()), B.stride(0), b_mn, M, Nn, K,
                                  P(C.data_ptr()), C.stride(0), ctypes.c_float(1.0), 0, P(stream))


x = torch.randn(N, 4 * H, device=dev).bfloat16()
w = torch.randn(4 * H, 4 * H, device=dev).bfloat16()
C = torch.empty(N, 4 * H, device=dev)
for name, M, Nn, K, am, bm in [("qkv fwd", N, 3 * H, H, 0, 0), ("ffn_in fwd", N, 4 * H, H, 0, 0),
                                ("ffn_out fwd", N, H, 4 * H, 0, 0), ("out fwd", N, H, H, 0, 0),
                                ("ffn_in dgrad", N, H, 4 * H, 0, 1), ("ffn_in wgrad", 4 * H, H, N, 1, 1)]:
    A = x if not am else x
    ms = timeit(gemm(x, am, w, bm, M, Nn, K, C))
    tf = 2.0 * M * Nn * K / ms / 1e9
    print(f"gemm {name:14s} {M}x{Nn}x{K}: {ms:8.3f} ms  {tf:7.1f} TFLOP/s")
del x, w, C

qkv = torch.randn(N, 3 * H, device=dev).bfloat16()
o = torch.empty(N, H, device=dev).bfloat16()
lse = torch.empty(heads, N, device=dev)
for tc in [1]:
    f = lambda: L.mgv_dev_attn_fwd(tc, P(qkv.data_ptr()), ctypes.c_int64(3 * H), P(qkv[:, H:].data_ptr()),
                                   ctypes.c_int64(3 * H), P(qkv[:, 2 * H:].data_ptr()), ctypes.c_int64(3 * H),
                                   P(o.data_ptr()), ctypes.c_int64(H), P(lse.data_ptr()), N, N, heads, hd, P(stream))
    ms = timeit(f, 3)
    fl = 4.0 * N * N * H
    print(f"attn fwd tc={tc} N={N}: {ms:8.3f} ms  {fl / ms / 1e9:7.1f} TFLOP/s")

# attention backward (self) at the same shape
dO = torch.randn(N, H, device=dev).bfloat16()
Dv = torch.empty(heads, N, device=dev)
dqkv = torch.empty(N, 3 * H, device=dev).bfloat16()
i64 = ctypes.c_int64
fb = lambda: L.mgv_dev_attn_bwd(1, P(qkv.data_ptr()), i64(3 * H), P(qkv[:, H:].data_ptr()), i64(3 * H),
                                P(qkv[:, 2 * H:].data_ptr()), i64(3 * H), P(o.data_ptr()), i64(H), P(lse.data_ptr()),
                                P(dO.data_ptr()), i64(H), P(Dv.data_ptr()), P(dqkv.data_ptr()), i64(3 * H),
                                P(dqkv[:, H:].data_ptr()), i64(3 * H), P(dqkv[:, 2 * H:].data_ptr()), i64(3 * H),
                                P(0), 1, N, N, heads, hd, P(stream))
ms = timeit(fb, 2)
fl = 8.0 * N * N * H
print(f"attn bwd tc N={N}: {ms:8.3f} ms  {fl / ms / 1e9:7.1f} TFLOP/s (algorithmic 8N^2H)")
