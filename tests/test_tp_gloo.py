"""The tensor-parallel decomposition on CPU (gloo, world_size 2): each rank computes one DiT block
(dit.cpp:279-313) from its Megatron shards (parallel.tp_shard) and the three partial
sums are all-reduced after attn.out, xattn.out and ffn.out; the result must equal the unsharded fp64
oracle block.  On the GPU the same shard map runs inside libmugv_b200.so (block_fwd_tp /
block_bwd_tp, checked against the oracle in test_tp_gpu.py with emulated ranks)."""
import math
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2510_17519_b200.parallel import tp_kind, tp_shard  # noqa: E402


def _case():
    cfg = O.DitConfig(depth=1, hidden=24, heads=4, text_dim=6, c_z=2, rope_split=(2, 2, 2))
    P = O.open_gates(O.init_dit_params(cfg, O.Rng(1)), 2)
    g = O.Rng(3)
    grids = [g.uniform_tensor((2, 4, 4, 2), -1, 1)]
    text = O.Rng(4).normal_tensor((3, 6))
    s = O.make_batch(grids, 0.0, O.Rng(5))[0]
    rows, tau, _, _ = O.masked_input(s)
    return cfg, P, text, rows, s.coords, tau


def tp_block_fwd(P, cfg, X, m, cos, sin, text, size, rank, allreduce):
    """One block from rank `rank`'s shards; allreduce(x) sums a partial over the TP group."""
    H, nh = cfg.hidden, cfg.heads
    Hr, nhr = H // size, nh // size
    S = {k: tp_shard(k, v, size, rank) for k, v in P.items() if k.startswith("dit.blk.0.")}
    b = "dit.blk.0."
    sh1, sc1, gt1, sh2, sc2, gt2 = [m[:, j * H:(j + 1) * H] for j in range(6)]
    n0, _ = O.rms_fwd(X)
    a = n0 * (1.0 + sc1) + sh1
    qkv = a @ S[b + "attn.qkv.w"].T + S[b + "attn.qkv.b"]  # (N, 3 Hr): q_r | k_r | v_r
    qn, _ = O.l2h_fwd(qkv[:, :Hr], nhr)
    kn, _ = O.l2h_fwd(qkv[:, Hr:2 * Hr], nhr)
    N = X.shape[0]
    qt = (qn.reshape(N, nhr, -1) * S[b + "attn.temp"][None, :, None]).reshape(N, Hr)
    Q = O.rope_apply(qt, cos, sin, nhr)
    K = O.rope_apply(kn, cos, sin, nhr)
    Oa, _ = O.mha_fwd(Q, K, qkv[:, 2 * Hr:], nhr)
    ao = allreduce(Oa @ S[b + "attn.out.w"].T) + P[b + "attn.out.b"]  # exchange 1
    X1 = X + ao * gt1
    n1, _ = O.rms_fwd(X1)
    cn = n1 * P[b + "xattn.prenorm.g"]
    cq = cn @ S[b + "xattn.q.w"].T + S[b + "xattn.q.b"]
    kv = text @ S[b + "xattn.kv.w"].T + S[b + "xattn.kv.b"]
    Ox, _ = O.mha_fwd(cq / math.sqrt(cfg.head_dim), kv[:, :Hr], kv[:, Hr:], nhr)
    co = allreduce(Ox @ S[b + "xattn.out.w"].T) + P[b + "xattn.out.b"]  # exchange 2 (before the post-norm)
    nco, _ = O.rms_fwd(co)
    X2 = X1 + nco * P[b + "xattn.postnorm.g"]
    n2, _ = O.rms_fwd(X2)
    f = n2 * (1.0 + sc2) + sh2
    h = O.silu(f @ S[b + "ffn.in.w"].T + S[b + "ffn.in.b"])
    ff = allreduce(h @ S[b + "ffn.out.w"].T) + P[b + "ffn.out.b"]  # exchange 3
    return X2 + ff * gt2


def _inputs(cfg, P, rows, coords, tau):
    X = rows @ P["dit.patch.w"].T + P["dit.patch.b"]
    gt, _ = O._mlp_fwd(O.sinusoid(O.TIMESTEP_SCALE * tau), P)
    gf, _ = O._mlp_fwd(O.sinusoid(np.array([8.0])), P)
    gb = (gt + gf) * P["dit.blk.0.gscale"]
    m = gb @ P["dit.mod.w"].T + P["dit.mod.b"]
    cos, sin = O.rope_tables(coords, cfg.rope_split)
    return X, m, cos, sin


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, P, text, rows, coords, tau = _case()
    X, m, cos, sin = _inputs(cfg, P, rows, coords, tau)

    def allreduce(x):
        t = torch.from_numpy(np.ascontiguousarray(x))
        dist.all_reduce(t)
        return t.numpy()

    out = tp_block_fwd(P, cfg, X, m, cos, sin, text, world, rank, allreduce)
    q.put((rank, out))
    dist.destroy_process_group()


def test_tp_shard_map_partitions():
    cfg = O.DitConfig(depth=1, hidden=24, heads=4, text_dim=6, c_z=2, rope_split=(2, 2, 2))
    P = O.init_dit_params(cfg, O.Rng(1))
    for size in (2, 4):
        for k, v in P.items():
            parts = [tp_shard(k, v, size, r) for r in range(size)]
            kind = tp_kind(k)
            if kind == "replicated":
                assert all(p is v for p in parts)
            elif kind == "cols":
                assert np.array_equal(np.concatenate(parts, axis=1), v)
            elif kind == "rows":
                assert np.array_equal(np.concatenate(parts, axis=0), v)
            else:  # chunked: every chunk is split evenly, so the union is a permutation of the rows
                C = 3 if "qkv" in k else 2
                cat = np.concatenate(parts, axis=0)
                R = v.shape[0] // C
                rs = R // size
                perm = [c * R + r * rs + j for r in range(size) for c in range(C) for j in range(rs)]
                assert np.array_equal(cat, v[perm])
    assert tp_kind("dit.blk.3.attn.qkv.w") == "chunked" and tp_kind("dit.mod.w") == "replicated"


def test_tp_emulated_ranks_match_oracle():
    """Single-process emulation: summing the per-rank partials reproduces the unsharded block."""
    cfg, P, text, rows, coords, tau = _case()
    X, m, cos, sin = _inputs(cfg, P, rows, coords, tau)
    _, taps, _ = O.velocity_fwd(P, cfg, rows, coords, tau, text, 8.0, keep=False)
    for size in (2, 4):
        # replace partials by sums progressively (each exchange depends on the previous ones)
        sums = []
        for step in range(3):
            outs = []
            for r in range(size):
                it = iter(sums)
                k = [0]

                def ar(x, it=it, k=k, outs=outs, r=r, step=step):
                    i = k[0]
                    k[0] += 1
                    if i < step:
                        return next(it)
                    if i == step:
                        outs.append(x)
                    return x
                tp_block_fwd(P, cfg, X, m, cos, sin, text, size, r, ar)
            sums.append(sum(outs))
        it = iter(sums)
        y = tp_block_fwd(P, cfg, X, m, cos, sin, text, size, 0, lambda x: next(it))
        assert np.abs(y - taps[1]).max() <= 1e-12 * max(1.0, np.abs(taps[1]).max())


def test_tp_gloo_world2():
    cfg, P, text, rows, coords, tau = _case()
    _, taps, _ = O.velocity_fwd(P, cfg, rows, coords, tau, text, 8.0, keep=False)
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        assert np.abs(outs[r] - taps[1]).max() <= 1e-12 * max(1.0, np.abs(taps[1]).max())
    assert np.array_equal(outs[0], outs[1])


def test_tp_storage_partitions_per_rank():
    """Sharded storage: per-rank parameter, gradient and AdamW bytes = replicated + sharded / P, and
    the 56-block 10B stack (configs[3]) at 10,920 tokens fits one B200 (180 GB) per rank at P = 4 and 8."""
    from paper_2510_17519_b200.capi import paper_config, plan_rank_bytes
    cfg = paper_config(56)
    b = {P: plan_rank_bytes(cfg, "bf16", P, 10920, 64, 2, True) for P in (1, 2, 4, 8)}
    # sharded parameters: qkv, out, xattn q/kv/out, ffn in/out per block (their biases and attn.temp too)
    H, L = 3456, 4096
    sharded = 56 * (3 * H * H + 3 * H + 24 + H * H + H * H + H + 2 * H * L + 2 * H + H * H + 4 * H * H + 4 * H + 4 * H * H)
    for P in (2, 4, 8):
        d_grad = b[1]["grads"] - b[P]["grads"]
        assert abs(d_grad - 4 * sharded * (1 - 1 / P)) < 4 * 64 * 56 * 12 * P, (P, d_grad)
        assert b[P]["adamw"] == 2 * b[P]["grads"]
        assert b[P]["workspace"] < b[1]["workspace"]
    tot = {P: sum(v.values()) for P, v in b.items()}
    assert tot[4] < 180e9 and tot[8] < 180e9 and tot[1] > 180e9, tot
