"""Tensor parallelism through the C ABI on one GPU: mgv_ctx_set_tp(size, 0, NULL) runs every TP rank's
shard views, per-rank GEMM/attention launches and the row-parallel partial sums of block_fwd_tp /
block_bwd_tp inside one context.  The result must match the fp64 oracle at the same
tolerances as the unsharded path, and the gradients come back in the reference row order."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.golden.make_golden import CASES, build_case
from tests.gpu_common import nerr, to_cfg, to_samples

pytestmark = pytest.mark.gpu
TOL = {"fp32": 1e-4, "bf16": 5e-2}


@pytest.mark.parametrize("name,size", [("hd144", 2), ("cfg0", 2), ("cfg0", 4)])
@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_tp_flow_step_parity(name, size, prec):
    from paper_2510_17519_b200.capi import Context
    cfg, P, text, samples = build_case(name, CASES[name])
    ref = O.flow_fwdbwd(P, cfg, samples, text, 8.0, grads=True)
    ctx = Context(0, prec)
    ctx.set_tp(size)
    ctx.upload(to_cfg(cfg), P)
    out = ctx.flow_step(to_samples(samples), text, 8.0, grads=True, velocity=True)
    errs = {"loss": abs(out["loss"] - ref["loss"]) / abs(ref["loss"]),
            "grad_norm": abs(out["grad_norm"] - O.grad_norm(ref["grads"])) / O.grad_norm(ref["grads"])}
    for i in range(len(samples)):
        errs[f"V{i}"] = nerr(out["V"][i], ref["V"][i])
    for k, g in ref["grads"].items():
        errs[k] = nerr(out["grads"][k], g)
    worst = max(errs, key=errs.get)
    print(f"tp{size} {name}/{prec}: worst {worst} {errs[worst]:.3e}")
    assert errs[worst] <= TOL[prec], (worst, errs[worst])


def test_tp_predict_velocity():
    from paper_2510_17519_b200.capi import Context
    cfg, P, text, samples = build_case("hd144", CASES["hd144"])
    s = samples[0]
    rows, tau, _, _ = O.masked_input(s)
    ctx = Context(0, "fp32")
    ctx.set_tp(2)
    ctx.upload(to_cfg(cfg), P)
    v = ctx.predict_velocity(rows, s.coords, s.dims, text, tau, 8.0)
    assert nerr(v, O.predict_velocity(P, cfg, rows, s.coords, tau, text, 8.0)) <= 1e-4


def test_tp_config_errors():
    from paper_2510_17519_b200.capi import Context, MugvError
    cfg, P, text, samples = build_case("hd144", CASES["hd144"])  # heads = 2
    ctx = Context(0, "fp32")
    ctx.set_tp(4)
    with pytest.raises(MugvError):
        ctx.upload(to_cfg(cfg), P)  # 4 does not divide 2 heads
    ctx2 = Context(0, "fp32")
    ctx2.upload(to_cfg(cfg), P)
    with pytest.raises(MugvError):
        ctx2.set_tp(2)  # after upload


# N not a multiple of P (45 tokens over 4 ranks) and a sample with fewer tokens than ranks (3 over 4): ranks
# own ceil(N/P) rows, the last owners fewer or none.
RAGGED = dict(CASES["cfg0"], grids=[(3, 6, 10), (1, 2, 6)], mask_prob=0.5, force_cond=[])


@pytest.mark.parametrize("name,size", [("hd144", 2), ("cfg0", 4), ("ragged", 4)])
@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_tp_peer_exchange(name, size, prec, monkeypatch):
    """The peer-memory exchange (row-parallel GEMM epilogue scatters into the owners' mailboxes, owners sum the
    slots in rank order and all-gather the rows; tp_peer.h) against the in-place accumulation of the partials in
    rank order (MGV_TP_EXCHANGE=nccl with emulated ranks): the same additions in the same order, so the step must
    be bit-identical; and against the fp64 oracle at the usual tolerance."""
    from paper_2510_17519_b200.capi import Context
    cfg, P, text, samples = build_case(name, RAGGED if name == "ragged" else CASES[name])
    outs = {}
    for mode in ["nccl", "peer"]:
        monkeypatch.setenv("MGV_TP_EXCHANGE", mode)
        ctx = Context(0, prec)
        ctx.set_tp(size)
        ctx.upload(to_cfg(cfg), P)
        outs[mode] = ctx.flow_step(to_samples(samples), text, 8.0, grads=True, velocity=True)
        ctx.close()
    a, b = outs["nccl"], outs["peer"]
    assert a["loss"] == b["loss"] and a["grad_norm"] == b["grad_norm"]
    for i in range(len(samples)):
        assert np.array_equal(a["V"][i], b["V"][i]), i
    for k in a["grads"]:
        assert np.array_equal(a["grads"][k], b["grads"][k]), k
    ref = O.flow_fwdbwd(P, cfg, samples, text, 8.0, grads=True)
    worst = max(nerr(b["grads"][k], g) for k, g in ref["grads"].items())
    worst = max([worst, abs(b["loss"] - ref["loss"]) / abs(ref["loss"])] +
                [nerr(b["V"][i], ref["V"][i]) for i in range(len(samples))])
    print(f"tp{size} peer {name}/{prec}: worst {worst:.3e}")
    assert worst <= TOL[prec]


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_planner_matches_a_real_context(prec):
    """mgv_plan_rank_bytes (the per-rank planner used for configs[3]) reproduces what a context actually allocates
    for the same step (tp = 1: one context is one rank)."""
    from paper_2510_17519_b200.capi import Context, plan_rank_bytes
    cfg, P, text, samples = build_case("hd144", CASES["hd144"])
    ctx = Context(0, prec)
    ctx.set_adamw(lr=1e-3)
    ctx.upload(to_cfg(cfg), P)
    s = samples[0]
    ctx.flow_step(to_samples([s]), text, 8.0)
    got = ctx.memory()
    plan = plan_rank_bytes(to_cfg(cfg), prec, 1, s.clean.shape[0], text.shape[0], 2, True)
    print(prec, got, plan)
    for k in ("params", "grads", "adamw", "workspace"):
        assert got[k] == plan[k], (k, got[k], plan[k])


def test_tp_with_dp_one_rank_communicator():
    """2-D parallelism path on one GPU: emulated TP = 2 plus the DP NCCL path (one-rank communicator: gradient and
    loss all-reduces of every step) gives bit-identical loss, gradients and AdamW weights to TP alone."""
    from paper_2510_17519_b200.capi import Context
    cfg, P, text, samples = build_case("hd144", CASES["hd144"])
    outs = []
    for dp in (False, True):
        c = Context(0, "bf16")
        if dp:
            c.set_dp(0, 1, Context.nccl_unique_id())
        c.set_tp(2)
        c.set_adamw(lr=1e-3, eps=1.0)
        c.upload(to_cfg(cfg), P)
        for _ in range(2):
            r = c.flow_step(to_samples(samples), text, 8.0, grads=True)
        outs.append((r, c.download()))
        c.close()
    (a, wa), (b, wb) = outs
    assert a["loss"] == b["loss"] and a["grad_norm"] == b["grad_norm"]
    for k in a["grads"]:
        assert np.array_equal(a["grads"][k], b["grads"][k]), k
        assert np.array_equal(wa[k], wb[k]), k


@pytest.mark.parametrize("name,size", [("hd144", 2), ("cfg0", 4), ("ragged", 4)])
def test_tp_bf16_payload(name, size, monkeypatch):
    """MGV_TP_PAYLOAD=bf16 (bf16 mode): the row-parallel epilogues write bf16 partials into the mailboxes and the
    owners all-gather bf16 sums (SURVEY 8(e)'s exchange bytes, half of fp32).  The step stays within the bf16
    tolerance of the oracle, differs from the fp32 payload only by that rounding, and is deterministic."""
    from paper_2510_17519_b200.capi import Context
    cfg, P, text, samples = build_case(name, RAGGED if name == "ragged" else CASES[name])
    monkeypatch.setenv("MGV_TP_EXCHANGE", "peer")
    outs = []
    for pay in ["fp32", "bf16", "bf16"]:
        monkeypatch.setenv("MGV_TP_PAYLOAD", pay)
        ctx = Context(0, "bf16")
        ctx.set_tp(size)
        ctx.upload(to_cfg(cfg), P)
        outs.append(ctx.flow_step(to_samples(samples), text, 8.0, grads=True, velocity=True))
        ctx.close()
    f32, b1, b2 = outs
    assert b1["loss"] == b2["loss"] and all(np.array_equal(b1["grads"][k], b2["grads"][k]) for k in b1["grads"])
    assert b1["loss"] != f32["loss"] or any(not np.array_equal(b1["V"][i], f32["V"][i]) for i in range(len(samples)))
    ref = O.flow_fwdbwd(P, cfg, samples, text, 8.0, grads=True)
    worst = max(nerr(b1["grads"][k], g) for k, g in ref["grads"].items())
    worst = max([worst, abs(b1["loss"] - ref["loss"]) / abs(ref["loss"])] +
                [nerr(b1["V"][i], ref["V"][i]) for i in range(len(samples))])
    print(f"tp{size} bf16 payload {name}: worst {worst:.3e}")
    assert worst <= TOL["bf16"]
