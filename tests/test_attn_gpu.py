"""tcgen05 flash attention (and the SIMT kernels) vs a plain torch fp32 reference of Tape::mha
(autodiff.cpp:755-843): per head softmax(q k^T) v, no scale, no mask."""
import ctypes

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def ref_attn(q, k, v, heads):
    Nq, H = q.shape
    hd = H // heads
    qh = q.float().view(Nq, heads, hd).transpose(0, 1)
    kh = k.float().view(-1, heads, hd).transpose(0, 1)
    vh = v.float().view(-1, heads, hd).transpose(0, 1)
    s = qh @ kh.transpose(1, 2)
    lse = torch.logsumexp(s, -1)
    o = torch.softmax(s, -1) @ vh
    return o.transpose(0, 1).reshape(Nq, H), lse


def make(Nq, Nk, heads, hd, unit, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    H = heads * hd
    qkv = torch.randn(max(Nq, Nk), 3 * H, device="cuda", generator=g)
    if unit:
        for j in range(2):
            x = qkv[:, j * H:(j + 1) * H].view(-1, heads, hd)
            x /= x.norm(dim=-1, keepdim=True)
            if j == 0:
                x *= 12.0
    qkv = qkv.bfloat16()
    return qkv[:Nq], qkv[:Nk], H


def call_fwd(tc, qbuf, kbuf, Nq, Nk, heads, hd):
    from paper_2510_17519_b200._lib import lib
    L = lib()
    L.mgv_dev_attn_fwd.restype = ctypes.c_int
    H = heads * hd
    o = torch.zeros(Nq, H, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(heads, Nq, device="cuda")
    P = ctypes.c_void_p
    rc = L.mgv_dev_attn_fwd(tc, P(qbuf.data_ptr()), ctypes.c_int64(qbuf.stride(0)), P(kbuf[:, H:].data_ptr()),
                            ctypes.c_int64(kbuf.stride(0)), P(kbuf[:, 2 * H:].data_ptr()), ctypes.c_int64(kbuf.stride(0)),
                            P(o.data_ptr()), ctypes.c_int64(H), P(lse.data_ptr()), Nq, Nk, heads, hd,
                            P(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    return o, lse


@pytest.mark.parametrize("tc", [1, 0])
@pytest.mark.parametrize("Nq,Nk,heads,hd,unit", [(300, 300, 2, 144, True), (1000, 64, 3, 144, False),
                                                 (256, 256, 2, 64, False), (2048, 2048, 2, 144, True),
                                                 (130, 400, 1, 128, False), (4096, 4096, 1, 144, False)])
def test_attn_fwd(tc, Nq, Nk, heads, hd, unit):
    qbuf, kbuf, H = make(Nq, Nk, heads, hd, unit, Nq + Nk + hd)
    o, lse = call_fwd(tc, qbuf, kbuf, Nq, Nk, heads, hd)
    ro, rl = ref_attn(qbuf[:, :H], kbuf[:, H:2 * H], kbuf[:, 2 * H:], heads)
    err = (o.float() - ro).abs().max().item() / ro.abs().max().item()
    lerr = (lse - rl).abs().max().item()
    print(f"tc={tc} {Nq}x{Nk} h{heads} hd{hd}: O err {err:.2e} lse err {lerr:.2e}")
    assert err < 2e-2 and lerr < 2e-2


def call_bwd(tc, qbuf, kbuf, o, lse, dO, Nq, Nk, heads, hd, q_splits=1):
    from paper_2510_17519_b200._lib import lib
    L = lib()
    H = heads * hd
    P = ctypes.c_void_p
    dq = torch.zeros(Nq, H, device="cuda", dtype=torch.bfloat16)
    dkv = torch.zeros(Nk, 2 * H, device="cuda", dtype=torch.bfloat16)
    Dv = torch.zeros(heads, Nq, device="cuda")
    part = torch.zeros(max(q_splits, 1) * heads * Nk * 2 * hd, device="cuda")
    i64 = ctypes.c_int64
    rc = L.mgv_dev_attn_bwd(tc, P(qbuf.data_ptr()), i64(qbuf.stride(0)), P(kbuf[:, H:].data_ptr()), i64(kbuf.stride(0)),
                            P(kbuf[:, 2 * H:].data_ptr()), i64(kbuf.stride(0)), P(o.data_ptr()), i64(H),
                            P(lse.data_ptr()), P(dO.data_ptr()), i64(H), P(Dv.data_ptr()), P(dq.data_ptr()), i64(H),
                            P(dkv.data_ptr()), i64(2 * H), P(dkv[:, H:].data_ptr()), i64(2 * H), P(part.data_ptr()),
                            q_splits, Nq, Nk, heads, hd, P(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    return dq, dkv[:, :H], dkv[:, H:]


# 1: the tcgen05 passes (dK/dV v8 + dQ v10); 0: the fp32 SIMT kernels
@pytest.mark.parametrize("tc", [1, 0])
@pytest.mark.parametrize("Nq,Nk,heads,hd,unit", [(300, 300, 2, 144, True), (1000, 64, 3, 144, False),
                                                 (256, 256, 2, 64, False), (2048, 2048, 2, 144, True),
                                                 (130, 400, 1, 128, False), (4000, 64, 2, 144, False)])
def test_attn_bwd(tc, Nq, Nk, heads, hd, unit):
    qbuf, kbuf, H = make(Nq, Nk, heads, hd, unit, 7 * Nq + Nk + hd)
    o, lse = call_fwd(1, qbuf, kbuf, Nq, Nk, heads, hd)
    g = torch.Generator(device="cuda").manual_seed(5)
    dO = torch.randn(Nq, H, device="cuda", generator=g).bfloat16()
    q = qbuf[:, :H].float().requires_grad_()
    k = kbuf[:, H:2 * H].float().requires_grad_()
    v = kbuf[:, 2 * H:].float().requires_grad_()
    ro, _ = ref_attn(q, k, v, heads)
    ro.backward(dO.float())
    dq, dk, dv = call_bwd(tc, qbuf, kbuf, o, lse, dO, Nq, Nk, heads, hd, q_splits=1 if tc else 4)
    errs = []
    for got, ref in [(dq, q.grad), (dk, k.grad), (dv, v.grad)]:
        errs.append((got.float() - ref).abs().max().item() / ref.abs().max().item())
    print(f"bwd tc={tc} {Nq}x{Nk} h{heads} hd{hd}: dq {errs[0]:.2e} dk {errs[1]:.2e} dv {errs[2]:.2e}")
    assert max(errs) < 3e-2
