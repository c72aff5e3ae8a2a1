"""forward_sample_rows / reverse_sample_rows (flowtrain.cpp:135-172) on device through mgv_sample_rows, against
the fp64 oracle sampler (pinned to the reference's in tests/test_oracle.py): Euler steps of the learned
probability-flow ODE with conditioned rows re-imposed, 4 steps."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.golden.make_golden import CASES, build_case
from tests.gpu_common import nerr, to_cfg

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec,tp", [("fp32", 1), ("fp32", 2), ("bf16", 1)])
@pytest.mark.parametrize("direction,cond", [(-1, False), (-1, True), (1, True)])
def test_sampler_parity(prec, tp, direction, cond):
    from paper_2510_17519_b200.capi import Context
    cfg, P, text, samples = build_case("hd144", CASES["hd144"])
    s = samples[0]
    N, D = s.coords.shape[0], 4 * cfg.c_z
    x0 = O.Rng(11).normal_tensor((N, D))
    cm = (s.coords[:, 0] == 0).astype(np.uint8) if cond else None
    cl = s.clean if cond else None
    ref = O.sample_rows(P, cfg, x0, s.coords, text, 8.0, 4, direction, cm, cl)
    ctx = Context(0, prec)
    if tp > 1:
        ctx.set_tp(tp)
    ctx.upload(to_cfg(cfg), P)
    got = ctx.sample_rows(x0, s.coords, s.dims, text, 4, direction, 8.0, cm, cl)
    err = nerr(got, ref)
    print(f"sampler {prec} tp{tp} dir{direction} cond{cond}: {err:.2e}")
    assert err <= (1e-4 if prec == "fp32" else 5e-2)
    if cond:  # conditioned rows carry the clean latents exactly
        assert np.array_equal(got[cm.astype(bool)], cl[cm.astype(bool)])


def test_sampler_errors():
    from paper_2510_17519_b200.capi import Context, InputError
    cfg, P, text, samples = build_case("tiny", CASES["tiny"])
    s = samples[0]
    ctx = Context(0, "fp32")
    ctx.upload(to_cfg(cfg), P)
    x0 = np.zeros((s.coords.shape[0], 4 * cfg.c_z))
    with pytest.raises(InputError):
        ctx.sample_rows(x0, s.coords, s.dims, text, 0)  # steps must be >= 1 (flowtrain.cpp:137)
    bad = np.zeros(s.coords.shape[0], dtype=np.uint8)
    bad[0] = 1  # one token of a unit: not frame-aligned (flowtrain.cpp:66-77)
    with pytest.raises(InputError):
        ctx.sample_rows(x0, s.coords, s.dims, text, 2, -1, 8.0, bad, x0)
