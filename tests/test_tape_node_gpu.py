"""mgv_velocity_graph: dit::velocity_rows_graph (dit.cpp:320-334) as one device tape node -- the forward with the
reference's taps (patch embedding, every block's residual output, the final projection, the velocity) and the
backward closure's vector-Jacobian product for an arbitrary upstream gradient dV -- against the oracle's
velocity_fwd / velocity_bwd (pinned to the reference by test_oracle.py), several distinct timesteps."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.golden.make_golden import CASES, build_case
from tests.gpu_common import nerr, to_cfg

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec,tol", [("fp32", 1e-4), ("bf16", 5e-2)])
def test_velocity_node_taps_and_vjp(prec, tol):
    from paper_2510_17519_b200.capi import Context
    cfg, P, text, samples = build_case("hd144", CASES["hd144"])
    s = samples[0]
    rows, tau, _, _ = O.masked_input(s)
    tau = tau.copy()
    tau[::3] = 0.25
    dV = O.Rng(11).normal_tensor(rows.shape)
    V, taps, c = O.velocity_fwd(P, cfg, rows, s.coords, tau, text, 8.0, keep=True)
    G = {k: np.zeros_like(v) for k, v in P.items()}
    O.velocity_bwd(P, cfg, c, dV, G)
    ctx = Context(0, prec)
    ctx.upload(to_cfg(cfg), P)
    out = ctx.velocity_graph(rows, s.coords, s.dims, text, tau, 8.0, taps=True, dV=dV)
    ctx.close()
    errs = {"V": nerr(out["V"], V)}
    assert len(out["taps"]) == len(taps) == cfg.depth + 3
    for i, (a, b) in enumerate(zip(out["taps"], taps)):
        errs[f"tap{i}"] = nerr(a, b)
    for k, g in G.items():
        errs[k] = nerr(out["grads"][k], g)
    worst = max(errs, key=errs.get)
    print(f"velocity node {prec}: worst {worst} {errs[worst]:.3e}")
    assert errs[worst] <= tol, (worst, errs[worst])
