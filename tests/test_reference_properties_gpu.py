"""The reference's own property tests for this path (SURVEY 8(c) pins), run through the C ABI on the GPU:

  zero-init head gives exactly 0, open gates give a deterministic non-zero output   test_dit.cpp:148-168, 518-535
  zero gates isolate tokens exactly; open gates mix them                            test_dit.cpp:171-203
  batch entries run exactly as batches of one                                       test_dit.cpp:205-222
  token-permutation equivariance                                                    test_dit.cpp:224-261
  velocity-model gradients match finite differences (fp32 mode)                     test_dit.cpp:490-516
  train-step determinism; abort on a non-finite loss without updating               test_flow.cpp:350-374

The reference checks exact equalities in fp64; where the device arithmetic makes an equality exact (gates,
zero heads, per-sample independence, repeat runs) the test demands it exactly, in both precisions."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.golden.make_golden import CASES
from tests.gpu_common import to_cfg, to_samples

pytestmark = pytest.mark.gpu
TINY = O.DitConfig(**CASES["tiny"]["cfg"])  # test_dit.cpp tiny_config: H12, 2 heads, depth 2, c_z 2
# the bf16 tensor-core mode needs head_dim % 16 == 0: the same tests at the smallest such shape
SMALL = O.DitConfig(depth=2, hidden=128, heads=2, text_dim=32, c_z=4, rope_split=(22, 22, 20))


def cfg_for(prec):
    return TINY if prec == "fp32" else SMALL


def ctx_with(P, prec):
    from paper_2510_17519_b200.capi import Context
    c = Context(0, prec)
    c.upload(to_cfg(cfg_for(prec)), P)
    return c


def tokens_grid(grid):
    rows, coords, dims = O.latent_rows(grid)
    return rows, coords, dims


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_zero_init_head_and_open_gates(prec):
    cfg = cfg_for(prec)
    r = O.Rng(131)
    P = O.init_dit_params(cfg, r)
    rows, coords, dims = tokens_grid(r.uniform_tensor((2, 2, 2, cfg.c_z), -1.0, 1.0))
    text = r.normal_tensor((1, cfg.text_dim))
    ts = np.full(rows.shape[0], 0.6)
    ctx = ctx_with(P, prec)
    v0 = ctx.predict_velocity(rows, coords, dims, text, ts)
    assert v0.shape == rows.shape and np.all(v0 == 0.0)
    tok = O.Rng(21).uniform_tensor((rows.shape[0], cfg.hidden), -1.0, 1.0)
    assert np.all(ctx.dit_forward(tok, coords, dims, text, np.full(rows.shape[0], 0.4)) == 0.0)
    ctx.close()
    ctx = ctx_with(O.open_gates(P, 17), prec)
    v1 = ctx.predict_velocity(rows, coords, dims, text, ts)
    v2 = ctx.predict_velocity(rows, coords, dims, text, ts)
    assert np.array_equal(v1, v2) and np.abs(v1).max() > 0.0
    ctx.close()


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_zero_gates_isolate_tokens(prec):
    cfg = cfg_for(prec)
    r = O.Rng(31)
    P = O.init_dit_params(cfg, r)
    P["dit.final.w"] = O.Rng(7).normal_tensor((cfg.hidden, cfg.hidden), 0.2)  # random head, zero gates
    _, coords, dims = tokens_grid(np.zeros((3, 2, 2, cfg.c_z)))
    N = coords.shape[0]
    tok = r.uniform_tensor((N, cfg.hidden), -1.0, 1.0)
    poked = tok.copy()
    poked[2] += 0.3  # token 2 only
    text = r.normal_tensor((2, cfg.text_dim))
    ts = np.full(N, 0.5)
    ctx = ctx_with(P, prec)
    base, pk = ctx.dit_forward(tok, coords, dims, text, ts), ctx.dit_forward(poked, coords, dims, text, ts)
    assert np.array_equal(base[:2], pk[:2])  # self-attention is the only cross-token path, multiplied by 0
    assert not np.array_equal(base[2], pk[2])
    ctx.close()
    ctx = ctx_with(O.open_gates(P, 5), prec)
    base, pk = ctx.dit_forward(tok, coords, dims, text, ts), ctx.dit_forward(poked, coords, dims, text, ts)
    assert np.abs(base[0] - pk[0]).max() > 0.0 and np.abs(base[1] - pk[1]).max() > 0.0
    ctx.close()


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_batch_entries_run_as_batches_of_one(prec):
    cfg = cfg_for(prec)
    r = O.Rng(41)
    P = O.open_gates(O.init_dit_params(cfg, r), 6)
    text = r.normal_tensor((3, cfg.text_dim))
    grids = [r.uniform_tensor((2, 2, 2, cfg.c_z), -1.0, 1.0), r.uniform_tensor((1, 4, 4, cfg.c_z), -1.0, 1.0)]
    s = O.make_batch(grids, 0.5, O.Rng(42))
    ctx = ctx_with(P, prec)
    joint = ctx.flow_step(to_samples(s), text, 8.0, velocity=True)
    for i in range(2):
        alone = ctx.flow_step(to_samples([s[i]]), text, 8.0, velocity=True)
        assert np.array_equal(joint["V"][i], alone["V"][0]), i
    ctx.close()


@pytest.mark.parametrize("prec,tol", [("fp32", 1e-5), ("bf16", 2e-2)])
def test_token_permutation_equivariance(prec, tol):
    cfg = cfg_for(prec)
    r = O.Rng(51)
    P = O.open_gates(O.init_dit_params(cfg, r), 8)
    text = r.normal_tensor((3, cfg.text_dim))
    _, coords, dims = tokens_grid(np.zeros((2, 4, 4, cfg.c_z)))
    N = coords.shape[0]
    tok = r.uniform_tensor((N, cfg.hidden), -1.0, 1.0)
    ts = np.where(np.arange(N) % 2 == 0, 0.3, 0.7)
    perm = np.arange(N)
    sr = O.Rng(17)
    for i in range(N - 1, 0, -1):  # the reference's Fisher-Yates with Rng(17).randint
        j = sr.randint(i + 1)
        perm[i], perm[j] = perm[j], perm[i]
    ctx = ctx_with(P, prec)
    out = ctx.dit_forward(tok, coords, dims, text, ts)
    out_s = ctx.dit_forward(tok[perm], coords[perm], dims, text, ts[perm])
    err = np.abs(out_s - out[perm]).max() / np.abs(out).max()
    print(f"{prec}: permutation equivariance error {err:.2e}")
    assert err < tol
    ctx.close()


def test_velocity_gradients_match_finite_differences():
    """Central differences of the flow loss (fp32 parity mode) against the device gradients, on the entries
    with the largest gradients of every parameter group (test_dit.cpp:490-516 checks < 1e-3)."""
    r = O.Rng(121)
    P = O.open_gates(O.init_dit_params(TINY, r), 13)
    text = r.normal_tensor((2, TINY.text_dim))
    s = O.make_batch([r.uniform_tensor((3, 2, 2, 2), -1.0, 1.0)], 0.0, O.Rng(5))
    s[0].cond = True
    ctx = ctx_with(P, "fp32")
    g = ctx.flow_step(to_samples(s), text, 8.0, grads=True)["grads"]
    worst = 0.0
    for name in ["dit.patch.w", "dit.blk.0.attn.qkv.w", "dit.blk.1.attn.temp", "dit.blk.0.ffn.in.w", "dit.mod.w",
                 "dit.blk.1.xattn.kv.w", "dit.gmlp.in.w", "dit.out.w"]:
        flat = g[name]
        idx = int(np.argmax(np.abs(flat)))
        h = 1e-3 * max(1.0, abs(float(P[name].ravel()[idx])))
        vals = []
        for sign in (1.0, -1.0):
            Q = {k: v.copy() for k, v in P.items()}
            Q[name].ravel()[idx] += sign * h
            ctx.upload(to_cfg(TINY), Q)
            vals.append(ctx.flow_step(to_samples(s), text, 8.0)["loss"])
        fd = (vals[0] - vals[1]) / (2 * h)
        rel = abs(fd - flat[idx]) / max(abs(flat[idx]), 1e-6)
        print(f"{name}[{idx}]: grad {flat[idx]:+.6e} fd {fd:+.6e} rel {rel:.1e}")
        worst = max(worst, rel)
    assert worst < 1e-3
    ctx.close()


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_train_step_determinism_and_nan_abort(prec):
    cfg = cfg_for(prec)
    from paper_2510_17519_b200.capi import Context, InputError, NumericError
    pr, tr = O.Rng(95), O.Rng(96)
    P = O.init_dit_params(cfg, pr)
    text = tr.normal_tensor((2, cfg.text_dim))
    s = O.make_batch([tr.uniform_tensor((2, 4, 4, cfg.c_z), -1.0, 1.0)], 0.5, O.Rng(97))
    runs = []
    for _ in range(2):
        c = Context(0, prec)
        c.set_adamw(lr=1e-3)
        c.upload(to_cfg(cfg), P)
        m = c.flow_step(to_samples(s), text, 8.0)
        runs.append((m, c.download()))
        c.close()
    (m1, w1), (m2, w2) = runs
    assert m1["loss"] == m2["loss"] and m1["grad_norm"] == m2["grad_norm"] and m1["grad_norm"] > 0.0
    for k in w1:
        assert np.array_equal(w1[k], w2[k]), k
    poisoned = {k: v.copy() for k, v in P.items()}
    poisoned["dit.patch.w"].ravel()[0] = np.nan
    c = Context(0, prec)
    c.set_adamw(lr=1e-3)
    c.upload(to_cfg(cfg), poisoned)
    before = c.download()
    with pytest.raises(NumericError):
        c.flow_step(to_samples(s), text, 8.0)
    assert c.adamw_steps() == 0  # the update was skipped, as the reference throws before AdamW
    after = c.download()
    for k in before:
        assert np.array_equal(before[k], after[k], equal_nan=True), k
    with pytest.raises(InputError):
        c.flow_step([], text, 8.0)
    c.close()
