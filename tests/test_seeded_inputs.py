"""The product's seeded-input helpers (the benchmark's SURVEY 8(d) inputs) reproduce the reference's Rng streams:
mgv_rng_uniform_fill = Rng(seed).uniform_tensor, mgv_make_flow_sample = make_batch's noise / t / mask draws, and
mgv_params_init = init_dit_params + open_gates (checked on the GPU: it uploads into a context)."""
import numpy as np
import pytest

from oracle import oracle as O


def test_rng_uniform_matches_oracle():
    from paper_2510_17519_b200.capi import rng_uniform
    a = rng_uniform(3, (2, 4, 6, 24), -1.0, 1.0)
    b = O.Rng(3).uniform_tensor((2, 4, 6, 24), -1.0, 1.0)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("mask_prob", [0.0, 1.0])
def test_make_flow_sample_matches_make_batch(mask_prob):
    from paper_2510_17519_b200.capi import make_flow_sample
    g = O.Rng(3).uniform_tensor((2, 4, 6, 24), -1.0, 1.0)
    s = O.make_batch([g], mask_prob, O.Rng(5))[0]
    noise, t, cond = make_flow_sample(5, s.clean.shape[0], 96, mask_prob)
    assert np.array_equal(noise, s.noise) and t == s.t and cond == s.cond


@pytest.mark.gpu
def test_params_init_matches_reference_init():
    from paper_2510_17519_b200.capi import Context
    from tests.gpu_common import to_cfg
    cfg = O.DitConfig(depth=2, hidden=288, heads=2, text_dim=64, c_z=24, rope_split=(48, 48, 48))
    gs = O.gate_std_for(288)
    P = O.open_gates(O.init_dit_params(cfg, O.Rng(1)), 2, gs, gs / 4)
    ctx = Context(0, "fp32")
    ctx.init_params(to_cfg(cfg), seed=1, gate_seed=2, gate_std=gs, gate_b_std=gs / 4)
    got = ctx.download()
    ctx.close()
    assert sorted(got) == sorted(P)
    for k in P:  # fp32 device masters of the reference's fp64 draws
        assert np.array_equal(got[k], P[k].astype(np.float32).astype(np.float64).ravel()), k
