"""The data-parallel decomposition on CPU (gloo, world_size 2): per-rank shards of the
batch, gradient all-reduce (sum) and the 1/B_global loss scaling reproduce the
single-process FlowTrainer::step gradients (flowtrain.cpp:257-279).  The per-rank
compute here is the fp64 oracle; on the GPU the same sharding feeds
libmugv_b200.so and the all-reduce is NCCL inside the library."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2510_17519_b200.parallel import shard, shard_indices  # noqa: E402


def _case():
    cfg = O.DitConfig(depth=1, hidden=12, heads=2, text_dim=6, c_z=2, rope_split=(2, 2, 2))
    P = O.open_gates(O.init_dit_params(cfg, O.Rng(1)), 2)
    g = O.Rng(3)
    grids = [g.uniform_tensor(s, -1, 1) for s in [(2, 4, 4, 2), (1, 4, 6, 2), (3, 2, 2, 2)]]
    text = O.Rng(4).normal_tensor((3, 6))
    samples = O.make_batch(grids, 0.5, O.Rng(5))
    samples[0].cond = True
    return cfg, P, text, samples


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, P, text, samples = _case()
    mine = shard(samples, rank, world)
    B = len(samples)
    G = {k: np.zeros_like(v) for k, v in P.items()}
    loss_sum = 0.0
    for s in mine:
        out = O.flow_fwdbwd(P, cfg, [s], text, 8.0, grads=True)  # l_b and grads of l_b (batch of one)
        loss_sum += out["loss"]
        for k in G:
            G[k] += out["grads"][k] / B  # local contribution to (1/B) sum_b dl_b
    names = sorted(G)
    flat = torch.tensor(np.concatenate([G[k].ravel() for k in names]))
    dist.all_reduce(flat)
    ls = torch.tensor([loss_sum], dtype=torch.float64)
    dist.all_reduce(ls)
    if rank == 0:
        q.put((ls.item() / B, flat.numpy()))
    dist.destroy_process_group()


def test_shard_indices_partition():
    for n in range(0, 9):
        for w in range(1, 4):
            got = sorted(i for r in range(w) for i in shard_indices(n, r, w))
            assert got == list(range(n))


def test_dp_world2_matches_single_process():
    cfg, P, text, samples = _case()
    ref = O.flow_fwdbwd(P, cfg, samples, text, 8.0, grads=True)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    loss, flat = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert abs(loss - ref["loss"]) < 1e-12 * abs(ref["loss"])
    names = sorted(ref["grads"])
    want = np.concatenate([ref["grads"][k].ravel() for k in names])
    assert np.abs(flat - want).max() <= 1e-12 * np.abs(want).max()
