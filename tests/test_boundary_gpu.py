"""The rest of the reference's value API at the boundary (dit.hpp:83-90): patchify, unpatchify and
global_embed through the C ABI, against the oracle (fp64 numpy restatement; the device runs IEEE-fp32 GEMMs
from the fp32 weight masters and the fp64 timestep MLP, so <= 1e-5 normwise in either precision mode)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.golden.make_golden import CASES, build_case
from tests.gpu_common import nerr, to_cfg

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_patchify_unpatchify_global_embed(prec):
    from paper_2510_17519_b200.capi import Context
    cfg, P, _, _ = build_case("hd144", CASES["hd144"])
    ctx = Context(0, prec)
    ctx.upload(to_cfg(cfg), P)
    grid = O.Rng(3).uniform_tensor((3, 6, 8, cfg.c_z), -1.0, 1.0)
    rows, coords, dims = O.latent_rows(grid)
    tok, co = ctx.patchify(grid)
    assert np.array_equal(co, coords)  # the index math is bit-exact
    ref_tok = rows @ P["dit.patch.w"].T + P["dit.patch.b"]
    assert nerr(tok, ref_tok) < 1e-5
    t2 = O.Rng(9).normal_tensor(tok.shape)
    back = ctx.unpatchify(t2, coords, dims)
    ref_rows = t2 @ P["dit.out.w"].T + P["dit.out.b"]
    assert nerr(back, O.rows_to_grid(ref_rows, coords, dims)) < 1e-5
    tau = np.where(np.arange(rows.shape[0]) % 3 == 0, 0.0, 0.37)
    g, bs = ctx.global_embed(tau, 8.0)
    assert nerr(g, O.global_embed(P, tau, 8.0)) < 1e-5
    for i in range(cfg.depth):
        assert np.array_equal(bs[i], P[f"dit.blk.{i}.gscale"].astype(np.float32).astype(np.float64))
    ctx.close()


def test_boundary_errors():
    from paper_2510_17519_b200.capi import Context, DimensionError, InputError
    cfg, P, _, _ = build_case("hd144", CASES["hd144"])
    ctx = Context(0, "fp32")
    ctx.upload(to_cfg(cfg), P)
    with pytest.raises(DimensionError):  # odd spatial dims (dit.cpp:95)
        ctx.patchify(np.zeros((1, 3, 4, cfg.c_z)))
    with pytest.raises(DimensionError):  # channels != c_z (dit.cpp:339-340)
        ctx.patchify(np.zeros((1, 2, 4, cfg.c_z + 1)))
    with pytest.raises(InputError):  # tau outside [0, 1] (dit.cpp:239-240)
        ctx.global_embed(np.array([0.5, 1.5]), 8.0)
    _, coords, dims = O.latent_rows(np.zeros((1, 2, 4, cfg.c_z)))
    with pytest.raises(DimensionError):  # duplicate coords (dit.cpp:132)
        ctx.unpatchify(np.zeros((2, cfg.hidden)), np.array([coords[0], coords[0]]), dims)
    ctx.close()
