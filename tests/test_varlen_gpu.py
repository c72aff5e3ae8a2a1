"""Varlen packing (BASELINE configs[4], mgv_ctx_set_varlen): a multi-sample flow step as one block-diagonal sequence.
Each sample's velocity (hence its loss) is bit-identical to the unpacked step -- the batch-of-one contract of
dit_forward_batch (test_dit.cpp:205-222) -- and the gradients match it up to summation order and the oracle at the
parity tolerance.  Sizes straddle the 128/256-row tiles, with first-frame and general conditioning mixed in."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.golden.make_golden import CASES, build_case
from tests.gpu_common import nerr, to_cfg, to_samples

pytestmark = pytest.mark.gpu


def mixed_batch():
    cfg, P, text, _ = build_case("hd144", CASES["hd144"])
    g = O.Rng(31)
    dims = [(3, 12, 20), (2, 30, 44), (1, 10, 8), (4, 16, 18)]  # N = 180, 660, 20, 288
    grids = [g.uniform_tensor((U, h, w, cfg.c_z), -1.0, 1.0) for (U, h, w) in dims]
    samples = O.make_batch(grids, 0.0, O.Rng(32))
    samples[1].cond = True  # first-frame
    units = samples[3].coords[:, 0]
    samples[3].mask = ((units == 1) | (units == 3)).astype(np.uint8)  # general unit-aligned mask
    samples[3].cond_latents = O.Rng(33).normal_tensor(samples[3].clean.shape)
    return cfg, P, text, samples


@pytest.mark.parametrize("prec,gtol", [("fp32", 1e-5), ("bf16", 2e-2)])
def test_packed_step_bit_equal_forward(prec, gtol):
    from paper_2510_17519_b200.capi import Context
    cfg, P, text, samples = mixed_batch()
    outs = []
    for packed in (False, True):
        ctx = Context(0, prec)
        ctx.set_varlen(packed)
        ctx.upload(to_cfg(cfg), P)
        outs.append(ctx.flow_step(to_samples(samples), text, 8.0, grads=True, velocity=True))
        ctx.close()
    a, b = outs
    for i in range(len(samples)):
        assert np.array_equal(a["V"][i], b["V"][i]), i  # the forward of every sample is bit-identical
    assert a["loss"] == b["loss"]
    worst = max(nerr(b["grads"][k], a["grads"][k]) for k in a["grads"])
    print(f"{prec}: packed vs sequential worst gradient {worst:.2e}")
    assert worst <= gtol


def test_packed_step_vs_oracle():
    from paper_2510_17519_b200.capi import Context
    cfg, P, text, samples = mixed_batch()
    ref = O.flow_fwdbwd(P, cfg, samples, text, 8.0, grads=True)
    ctx = Context(0, "fp32")
    ctx.set_varlen(True)
    ctx.upload(to_cfg(cfg), P)
    out = ctx.flow_step(to_samples(samples), text, 8.0, grads=True, velocity=True)
    ctx.close()
    errs = {"loss": abs(out["loss"] - ref["loss"]) / abs(ref["loss"])}
    for i in range(len(samples)):
        errs[f"V{i}"] = nerr(out["V"][i], ref["V"][i])
    for k, g in ref["grads"].items():
        errs[k] = nerr(out["grads"][k], g)
    worst = max(errs, key=errs.get)
    assert errs[worst] <= 1e-4, (worst, errs[worst])


def test_packed_step_under_tensor_parallelism():
    """Varlen packing composes with (emulated) TP = 2: every sample's velocity bit-identical to the unpacked TP
    step, gradients within 1e-5 (fp32)."""
    from paper_2510_17519_b200.capi import Context
    cfg, P, text, samples = mixed_batch()
    outs = []
    for packed in (False, True):
        ctx = Context(0, "fp32")
        ctx.set_tp(2)
        ctx.set_varlen(packed)
        ctx.upload(to_cfg(cfg), P)
        outs.append(ctx.flow_step(to_samples(samples), text, 8.0, grads=True, velocity=True))
        ctx.close()
    a, b = outs
    for i in range(len(samples)):
        assert np.array_equal(a["V"][i], b["V"][i]), i
    assert max(nerr(b["grads"][k], a["grads"][k]) for k in a["grads"]) <= 1e-5
