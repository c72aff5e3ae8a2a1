"""The SPEC-only operators of the path through the C ABI: fused_modulate and
apply_rope3d (SPEC.md:168-176 = Tape::rope3d, autodiff.cpp:849-898).

fused_modulate's oracle is the composed three-step reference in the same precision and order (numpy fp64 for
the host op, torch fp32 elementwise kernels for the device op): bit-exact, as SPEC.md:620,630 require.
apply_rope3d is compared bit-for-bit with the compiled reference (oracle/_ref, Tape::rope3d forward and its
backward's inverse rotation), plus the SPEC's own examples."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _ctx():
    from paper_2510_17519_b200.capi import Context
    return Context(0, "fp32")


def test_fused_modulate_bit_exact():
    ctx = _ctx()
    rng = np.random.default_rng(7)
    rows, cols = 1000, 1000  # 10^6 elements
    x, res = rng.standard_normal((rows, cols)), rng.standard_normal((rows, cols))
    for shape in [(cols,), (1,), (rows, cols)]:  # per channel, scalar, full
        b, sc, sh = (rng.standard_normal(shape) for _ in range(3))
        ref = res + ((x + b) * (1.0 + sc) + sh)  # composed: bias, modulation, residual
        out = ctx.fused_modulate(x, b, sc, sh, res)
        assert np.array_equal(out, ref), shape
    z = np.zeros(cols)
    assert np.array_equal(ctx.fused_modulate(x, z, z, z, res), res + x)
    sh = rng.standard_normal(cols)
    zz = np.zeros((rows, cols))
    assert np.array_equal(ctx.fused_modulate(zz, z, rng.standard_normal(cols), sh, zz), np.broadcast_to(sh, zz.shape))
    ctx.close()


def test_fused_modulate_errors():
    from paper_2510_17519_b200.capi import DimensionError
    ctx = _ctx()
    x = np.ones((4, 6))
    with pytest.raises(DimensionError):  # broadcast mismatch
        ctx.fused_modulate(x, np.ones(5), np.ones(6), np.ones(6), x)
    assert ctx.fused_modulate(np.ones((0, 6)), np.ones(6), np.ones(6), np.ones(6), np.ones((0, 6))).shape == (0, 6)
    ctx.close()


def test_fused_modulate_device_f32():
    import torch
    ctx = _ctx()
    g = torch.Generator(device="cuda").manual_seed(3)
    rows, cols = 57600, 3456  # one (N, H) residual-stream tensor at the 720p shape
    x = torch.randn(rows, cols, device="cuda", generator=g)
    res = torch.randn(rows, cols, device="cuda", generator=g)
    b, sc, sh = (torch.randn(cols, device="cuda", generator=g) for _ in range(3))
    out = torch.empty_like(x)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    ctx.dev_fused_modulate_f32(x, b, sc, sh, res, out)
    ref = res + ((x + b) * (1.0 + sc) + sh)  # separate torch kernels: no contraction across the steps
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    # one traversal: 12 bytes of HBM traffic per element (read x, residual; write out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        ctx.dev_fused_modulate_f32(x, b, sc, sh, res, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"fused_modulate f32 {rows}x{cols}: {ms:.3f} ms, {12.0 * rows * cols / ms / 1e6:.0f} GB/s")
    ctx.close()


def _coords(N, rng, lo=0, hi=40):
    return rng.integers(lo, hi, size=(N, 3)).astype(np.int32)


@pytest.mark.skipif(O.ref_lib() is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("split,heads", [((48, 48, 48), 3), ((22, 22, 20), 4), ((4, 6, 6), 2), ((0, 8, 8), 1)])
def test_apply_rope3d_bit_exact_vs_reference(split, heads):
    import ctypes
    L = O.ref_lib()
    ctx = _ctx()
    rng = np.random.default_rng(sum(split) + heads)
    N = 300
    x = rng.standard_normal((N, heads * sum(split)))
    co = _coords(N, rng, -5, 60)
    sp = (ctypes.c_int * 3)(*split)
    for inverse in (0, 1):
        ref = np.empty_like(x)
        assert L.ref_rope3d(x.ctypes.data, N, heads, sp, co.ctypes.data, 10000.0, inverse, ref.ctypes.data) == 0
        out = ctx.apply_rope3d(x, co, split, heads, inverse=bool(inverse))
        assert np.array_equal(out, ref), (split, inverse)
    ctx.close()


def test_apply_rope3d_properties():
    from paper_2510_17519_b200.capi import ConfigError
    ctx = _ctx()
    rng = np.random.default_rng(11)
    split, heads, N = (48, 48, 48), 2, 64
    x = rng.standard_normal((N, heads * 144))
    zero = np.zeros((N, 3), np.int32)
    assert np.array_equal(ctx.apply_rope3d(x, zero, split, heads), x)  # zero angles
    co = _coords(N, rng)
    y = ctx.apply_rope3d(x, co, split, heads)
    yh, xh = y.reshape(N, heads, 144), x.reshape(N, heads, 144)
    assert np.allclose(np.linalg.norm(yh, axis=2), np.linalg.norm(xh, axis=2), rtol=1e-12)  # norm preserved
    assert np.allclose(ctx.apply_rope3d(y, co, split, heads, inverse=True), x, atol=1e-12)
    # relative position: <rope(q, p1 + d), rope(k, p2 + d)> == <rope(q, p1), rope(k, p2)>
    q, k = rng.standard_normal((N, 144)), rng.standard_normal((N, 144))
    p1, p2, d = _coords(N, rng), _coords(N, rng), rng.integers(0, 30, size=(1, 3)).astype(np.int32)
    a = np.sum(ctx.apply_rope3d(q, p1 + d, split, 1) * ctx.apply_rope3d(k, p2 + d, split, 1), 1)
    b = np.sum(ctx.apply_rope3d(q, p1, split, 1) * ctx.apply_rope3d(k, p2, split, 1), 1)
    assert np.max(np.abs(a - b)) < 1e-5
    with pytest.raises(ConfigError):  # odd slice (autodiff.cpp:874-876)
        ctx.apply_rope3d(np.ones((2, 15)), np.zeros((2, 3), np.int32), (5, 6, 4), 1)
    ctx.close()
