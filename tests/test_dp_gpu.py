"""Data parallelism through the library (not the oracle): the batch split over `world` ranks, each rank's
context computing its share of FlowTrainer::step (mgv_ctx_set_dp without a communicator: loss and gradients scaled
by 1 / global batch, unreduced), sums over the ranks to the single-context step -- the decomposition the NCCL
all-reduce performs on a real multi-GPU run (flowtrain.cpp:263-273 loss scaling; every rank holds the same number
of samples, global batch = n_local x world)."""
import numpy as np
import pytest

from tests.golden.make_golden import CASES, build_case
from tests.gpu_common import nerr, to_cfg, to_samples
from tests.test_varlen_gpu import mixed_batch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("prec,tol", [("fp32", 1e-6), ("bf16", 1e-5)])
def test_dp_shares_sum_to_the_global_step(world, prec, tol):
    from paper_2510_17519_b200.capi import Context
    cfg, P, text, samples = mixed_batch()  # 4 samples of 180 / 660 / 20 / 288 tokens, mixed conditioning
    full = Context(0, prec)
    full.upload(to_cfg(cfg), P)
    ref = full.flow_step(to_samples(samples), text, 8.0, grads=True)
    full.close()
    shards = [samples[r::world] for r in range(world)]
    loss, grads = 0.0, None
    for r, shard in enumerate(shards):
        ctx = Context(0, prec)
        ctx.set_dp(r, world, None)
        ctx.upload(to_cfg(cfg), P)
        out = ctx.flow_step(to_samples(shard), text, 8.0, grads=True)
        ctx.close()
        loss += out["loss"]  # this rank's sum of l_b / (n_local * world)
        grads = out["grads"] if grads is None else {k: grads[k] + v for k, v in out["grads"].items()}
    assert abs(loss - ref["loss"]) <= 1e-12 * abs(ref["loss"]) + 1e-15
    worst = max(nerr(grads[k], g) for k, g in ref["grads"].items())
    print(f"world {world} {prec}: summed shares vs global step, worst gradient {worst:.2e}")
    assert worst <= tol
