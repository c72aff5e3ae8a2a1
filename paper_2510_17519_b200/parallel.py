"""Host-side data-parallel plumbing for the flow step.

Samples are independent (dit.hpp:97-100), so data parallelism shards the batch:
rank r of W owns samples r, r+W, r+2W, ...  Each rank runs forward + backward
on its shard; gradients are summed across ranks (NCCL all-reduce inside
libmugv_b200.so, mgv_ctx_set_dp) and the loss is the global mean
L = (1/B_global) sum_b l_b (flowtrain.cpp:273).  No collective touches the
data path itself.
"""
from __future__ import annotations


def shard_indices(n_samples: int, rank: int, world: int) -> list[int]:
    """Round-robin sample ownership (deterministic, covers every sample exactly once)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return list(range(rank, n_samples, world))


def shard(samples: list, rank: int, world: int) -> list:
    return [samples[i] for i in shard_indices(len(samples), rank, world)]


def global_batch(local_counts: list[int]) -> int:
    return int(sum(local_counts))
