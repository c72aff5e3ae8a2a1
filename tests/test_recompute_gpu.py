"""Per-block activation recompute (mgv_ctx_set_recompute; SURVEY 8(d) config 4's option for deep stacks at 57,600
tokens): the training step keeps only every block's input rows and re-runs each block's forward inside the backward.
Same kernels on the same inputs, so loss, velocity and every gradient must be bit-identical to keeping the
activations -- unsharded, under emulated TP, and with varlen packing -- while the workspace shrinks to one block's
activations (the planner and a live context agree)."""
import numpy as np
import pytest

from tests.golden.make_golden import CASES, build_case
from tests.gpu_common import to_cfg, to_samples

pytestmark = pytest.mark.gpu

DEEP = dict(CASES["hd144"], cfg=dict(CASES["hd144"]["cfg"], depth=4))


def _step(spec, prec, recompute, tp=1, varlen=False):
    from paper_2510_17519_b200.capi import Context
    cfg, P, text, samples = build_case("hd144", spec)
    ctx = Context(0, prec)
    if tp > 1:
        ctx.set_tp(tp)
    ctx.set_recompute(recompute)
    ctx.set_varlen(varlen)
    ctx.upload(to_cfg(cfg), P)
    out = ctx.flow_step(to_samples(samples), text, 8.0, grads=True, velocity=True)
    out["memory"] = ctx.memory()
    ctx.close()
    return out, cfg


def _same(a, b):
    assert a["loss"] == b["loss"] and a["grad_norm"] == b["grad_norm"]
    for va, vb in zip(a["V"], b["V"]):
        assert np.array_equal(va, vb)
    for k in a["grads"]:
        assert np.array_equal(a["grads"][k], b["grads"][k]), k


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("tp,varlen", [(1, False), (2, False), (1, True)])
def test_recompute_bit_identical(prec, tp, varlen):
    keep, _ = _step(DEEP, prec, False, tp, varlen)
    rec, _ = _step(DEEP, prec, True, tp, varlen)
    _same(keep, rec)
    assert rec["memory"]["workspace"] < keep["memory"]["workspace"]


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_recompute_planner_matches_context(prec):
    """mgv_plan_rank_bytes(train = 3) reproduces a recomputing context's allocations for the same one-sample step."""
    from paper_2510_17519_b200.capi import Context, plan_rank_bytes
    cfg, P, text, samples = build_case("hd144", DEEP)
    ctx = Context(0, prec)
    ctx.set_adamw(lr=1e-3)
    ctx.set_recompute(True)
    ctx.upload(to_cfg(cfg), P)
    s = samples[0]
    ctx.flow_step(to_samples([s]), text, 8.0)
    got = ctx.memory()
    ctx.close()
    plan = plan_rank_bytes(to_cfg(cfg), prec, 1, s.clean.shape[0], text.shape[0], 2, True, recompute=True)
    keep = plan_rank_bytes(to_cfg(cfg), prec, 1, s.clean.shape[0], text.shape[0], 2, True)
    for k in ("params", "grads", "adamw", "workspace"):
        assert got[k] == plan[k], (k, got[k], plan[k])
    assert plan["workspace"] < keep["workspace"]
