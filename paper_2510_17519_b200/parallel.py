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


# ---------------------------------------------------------------- tensor parallel (Megatron head/column)
# Shard map of SURVEY 8(e).  Rank r of P owns heads [r nh/P, (r+1) nh/P): its rows of each chunk of the
# chunked projections (attn.qkv: q|k|v, xattn.kv: k|v -- the chunk layout of expansion.cpp:143-180) and
# its entries of attn.temp; its rows of xattn.q and ffn.in (column-parallel); its columns of the
# row-parallel attn.out / xattn.out / ffn.out.  Everything else is replicated.  libmugv_b200.so applies
# the same map (rank-major row permutation at upload, model.cu tp_row_chunks / block_fwd_tp).
_TP_CHUNKED = {"attn.qkv.w": 3, "attn.qkv.b": 3, "xattn.kv.w": 2, "xattn.kv.b": 2}
_TP_ROWS = ("attn.temp", "xattn.q.w", "xattn.q.b", "ffn.in.w", "ffn.in.b")
_TP_COLS = ("attn.out.w", "xattn.out.w", "ffn.out.w")


def tp_kind(name: str) -> str:
    """'chunked', 'rows', 'cols' or 'replicated' for a dit.* parameter name."""
    if not name.startswith("dit.blk."):
        return "replicated"
    leaf = name.split(".", 3)[3]
    if leaf in _TP_CHUNKED:
        return "chunked"
    if leaf in _TP_ROWS:
        return "rows"
    if leaf in _TP_COLS:
        return "cols"
    return "replicated"


def tp_shard(name: str, arr, size: int, rank: int):
    """Rank `rank`'s slice of parameter `name` (reference row order within the slice)."""
    import numpy as np
    if size < 1 or not (0 <= rank < size):
        raise ValueError("bad tensor-parallel rank/size")
    kind = tp_kind(name)
    if kind == "replicated":
        return arr
    if kind == "cols":
        c = arr.shape[1] // size
        return arr[:, rank * c:(rank + 1) * c]
    if kind == "rows":
        r = arr.shape[0] // size
        return arr[rank * r:(rank + 1) * r]
    C = _TP_CHUNKED[name.split(".", 3)[3]]
    R = arr.shape[0] // C
    rs = R // size
    return np.concatenate([arr[c * R + rank * rs:c * R + (rank + 1) * rs] for c in range(C)], axis=0)
