"""The per-rank memory planner (mgv_plan_rank_bytes, the runtime's own workspace layout in measure mode; no device
needed) for the deep-stack configurations of BASELINE configs[3] / SURVEY 8(d) config 4: tensor parallelism
partitions the parameters, gradients and moments, per-block recompute shrinks the workspace to one block's
activations plus the kept inputs, and the full 56-block stack at 57,600 tokens fits a 180 GB B200 per rank from
TP 2 with recompute (at 10,920 tokens from TP 4 without it)."""
import pytest

from paper_2510_17519_b200.capi import paper_config, plan_rank_bytes

GB = 1e9
B200 = 180 * GB


def total(d):
    return sum(d.values())


@pytest.mark.parametrize("N", [10920, 57600])
def test_tp_partitions_state(N):
    cfg = paper_config(depth=56)  # the blocks dominate; the shared modulation weight and heads stay replicated
    one = plan_rank_bytes(cfg, "bf16", 1, N, 64)
    for p in (2, 4, 8):
        r = plan_rank_bytes(cfg, "bf16", p, N, 64)
        for k in ("params", "grads", "adamw"):
            assert r[k] < one[k] / p * 1.2, (p, k)  # sharded matrices dominate; norms/gains replicated
        assert r["workspace"] < one["workspace"]


@pytest.mark.parametrize("tp", [1, 2, 8])
def test_recompute_shrinks_workspace(tp):
    cfg = paper_config(depth=8)
    keep = plan_rank_bytes(cfg, "bf16", tp, 57600, 64)
    rec = plan_rank_bytes(cfg, "bf16", tp, 57600, 64, recompute=True)
    assert rec["workspace"] < keep["workspace"] / 3
    for k in ("params", "grads", "adamw", "exchange"):
        assert rec[k] == keep[k]


def test_full_stack_fits():
    cfg = paper_config(depth=56)
    assert total(plan_rank_bytes(cfg, "bf16", 2, 57600, 64, recompute=True)) < B200
    assert total(plan_rank_bytes(cfg, "bf16", 1, 57600, 64, recompute=True)) > B200
    assert total(plan_rank_bytes(cfg, "bf16", 4, 10920, 64)) < B200
    assert total(plan_rank_bytes(cfg, "bf16", 2, 10920, 64)) > B200
