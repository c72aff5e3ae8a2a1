"""The fusions against the kernels they replace -- the QKV projection with the QK-L2-norm x temperature + 3-D RoPE
in its epilogue (EpiQKNormRope, BN = head_dim; replaces GEMM + qk_norm_rope_vec), the post-norm residual with the
FFN's modulated RMSNorm (replaces postnorm_resid_vec + rms_fwd_vec), and the attention operands' transposes written
by the producing GEMM epilogues (Q^T / K^T / V^T / q'^T / dO^T; replaces five transpose_bf16 launches per step):
the whole bf16 training step (loss, velocity, every gradient) must be bit-identical with the fusions on and off.  Parity of the
unfused path against the oracle is test_parity_gpu.py / test_parity_golden_gpu.py; this pins the fusions to it
exactly.

Cases cover both GEMM kernels (<= 128 tokens: the 1-CTA kernel; more: the CTA-pair kernel), tiles straddling
the token count, head_dim 64 and 144, the 10B width (24 heads), and emulated tensor parallelism (per-rank
QKLayout with compact leading dimensions)."""
import numpy as np
import pytest

from tests.golden.make_golden import CASES, LONG_CASES, build_case
from tests.gpu_common import to_cfg, to_samples

pytestmark = pytest.mark.gpu

EXTRA = {
    # 3 x 10 x 12 = 360 tokens per sample: CTA-pair tiles with a partial last pair, two samples
    "hd144_360": dict(cfg=dict(depth=1, hidden=288, heads=2, text_dim=64, c_z=24, rope_split=(48, 48, 48)),
                      grids=[(3, 20, 24), (2, 18, 10)], L=8, mask_prob=0.0, force_cond=[0],
                      gate_std=CASES["hd144"]["gate_std"], full=False),
}


def _step(name, spec, fused, tp=1):
    """fused: bit mask of mgv_dev_set_fusions (1 QKV epilogue, 2 post-norm + modulated RMSNorm, 4 transposes)"""
    from paper_2510_17519_b200._lib import lib
    from paper_2510_17519_b200.capi import Context
    cfg, P, text, samples = build_case(name, spec)
    lib().mgv_dev_set_fusions(fused)
    try:
        ctx = Context(0, "bf16")
        if tp > 1:
            ctx.set_tp(tp)
        ctx.upload(to_cfg(cfg), P)
        out = ctx.flow_step(to_samples(samples), text, 8.0, grads=True, velocity=True)
        ctx.close()
    finally:
        lib().mgv_dev_set_fusions(7)
    return out


def _same(a, b):
    assert a["loss"] == b["loss"]
    assert a["grad_norm"] == b["grad_norm"]
    for va, vb in zip(a["V"], b["V"]):
        assert np.array_equal(va, vb)
    for k in a["grads"]:
        assert np.array_equal(a["grads"][k], b["grads"][k]), k


@pytest.mark.parametrize("name", ["cfg0", "hd144", "hd144_360", "w10b"])
@pytest.mark.parametrize("mask", [1, 2, 3, 5, 7])
def test_fusions_bit_identical(name, mask):
    spec = dict(CASES, **LONG_CASES, **EXTRA)[name]
    _same(_step(name, spec, mask), _step(name, spec, 0))


@pytest.mark.parametrize("tp", [2])
def test_fusions_bit_identical_tp(tp):
    _same(_step("hd144_360", EXTRA["hd144_360"], 7, tp), _step("hd144_360", EXTRA["hd144_360"], 0, tp))
