"""Parity at the benchmark's full size (BASELINE configs[2]: 10B dims, 720p/5s latent 16x90x160 -> 57,600
tokens), where the fp64 oracle cannot run (its probabilities tensor alone would be 637 GB):

1. the 2x2 patch index math at the full grid, bit-exact against the oracle's C restatement;
2. the tcgen05 attention at N = 57,600, 24 heads x 144: sampled query rows (O, lse, dQ) and sampled key rows
   (dK, dV) against an fp64 evaluation of Tape::mha and its backward (autodiff.cpp:755-843) on the same
   bf16 inputs;
3. the whole FlowTrainer::step at 57,600 tokens: the bf16 tensor-core mode against the IEEE-fp32 parity mode
   (itself pinned to the oracle at small sizes, tests/test_parity_gpu.py), within the bf16 tolerance, and
   bit-identical repeated runs."""
import numpy as np
import pytest

from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

N_FULL = 57600
GRID = (16, 90, 160, 24)  # (U, h, w, c_z): 16 x 45 x 80 tokens after 2x2 patchify


def test_patch_index_math_full_grid():
    from paper_2510_17519_b200.capi import Context
    g = O.Rng(3).uniform_tensor(GRID, -1.0, 1.0)
    rows_o, coords_o, dims_o = O.latent_rows(g)
    ctx = Context(0, "bf16")
    rows, coords = ctx.latent_rows(g)
    assert rows.shape == (N_FULL, 96) and tuple(dims_o) == (16, 45, 80)
    assert np.array_equal(coords, coords_o) and rows.tobytes() == rows_o.tobytes()
    back = ctx.rows_to_grid(rows, coords, dims_o, 24)
    assert back.tobytes() == g.tobytes()
    ctx.close()


def _attn_inputs(N, heads, hd, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    H = heads * hd
    qkv = torch.randn(N, 3 * H, device="cuda", generator=g)
    for j in range(2):  # unit-norm q / k per head, temperature ~ 10 (what the QK-norm produces)
        x = qkv[:, j * H:(j + 1) * H].view(N, heads, hd)
        x /= x.norm(dim=-1, keepdim=True)
        if j == 0:
            x *= 10.0
    return qkv.bfloat16(), H


def test_attention_sampled_rows_57600():
    from tests.test_attn_gpu import call_bwd, call_fwd
    heads, hd, N = 24, 144, N_FULL
    qkv, H = _attn_inputs(N, heads, hd, 11)
    o, lse = call_fwd(1, qkv, qkv, N, N, heads, hd)
    g = torch.Generator(device="cuda").manual_seed(12)
    dO = (torch.randn(N, H, device="cuda", generator=g) * 0.1).bfloat16()
    dq, dk, dv = call_bwd(1, qkv, qkv, o, lse, dO, N, N, heads, hd)
    rows = torch.randperm(N, generator=torch.Generator().manual_seed(13))[:32].cuda()
    keys = torch.randperm(N, generator=torch.Generator().manual_seed(14))[:16].cuda()
    worst = {}
    for h in (0, 7, 23):
        c = slice(h * hd, (h + 1) * hd)
        Q = qkv[:, c].double()
        K = qkv[:, H + h * hd:H + (h + 1) * hd].double()
        V = qkv[:, 2 * H + h * hd:2 * H + (h + 1) * hd].double()
        dOh = dO[:, c].double()
        # every query row's lse and D = dO . O (fp64, in chunks): needed for the key-row gradients
        lse_all = torch.empty(N, dtype=torch.float64, device="cuda")
        D_all = torch.empty(N, dtype=torch.float64, device="cuda")
        for a in range(0, N, 2048):
            s = Q[a:a + 2048] @ K.T
            lse_all[a:a + 2048] = torch.logsumexp(s, -1)
            oo = torch.softmax(s, -1) @ V
            D_all[a:a + 2048] = (dOh[a:a + 2048] * oo).sum(-1)
        # query rows: O, lse, dQ = sum_j P_ij (dP_ij - D_i) k_j   (autodiff.cpp:811-823)
        s = Q[rows] @ K.T
        p = torch.softmax(s, -1)
        o_ref = p @ V
        dP = dOh[rows] @ V.T
        dq_ref = (p * (dP - D_all[rows, None])) @ K
        # key rows: dV_j = sum_i P_ij dO_i, dK_j = sum_i P_ij (dP_ij - D_i) q_i
        sk = Q @ K[keys].T  # (N, 16)
        pk = torch.exp(sk - lse_all[:, None])
        dv_ref = pk.T @ dOh
        dPk = dOh @ V[keys].T
        dk_ref = (pk * (dPk - D_all[:, None])).T @ Q
        for name, got, ref in [("O", o[rows][:, c], o_ref), ("dQ", dq[rows][:, c], dq_ref),
                               ("dK", dk[keys][:, c], dk_ref), ("dV", dv[keys][:, c], dv_ref)]:
            e = ((got.double() - ref).abs().max() / ref.abs().max()).item()
            worst[name] = max(worst.get(name, 0.0), e)
        worst["lse"] = max(worst.get("lse", 0.0), (lse[h, rows].double() - lse_all[rows]).abs().max().item())
    print("57.6K attention, sampled rows vs fp64:", {k: f"{v:.2e}" for k, v in worst.items()})
    assert worst["O"] < 2e-2 and worst["lse"] < 2e-2
    assert worst["dQ"] < 3e-2 and worst["dK"] < 3e-2 and worst["dV"] < 3e-2


def test_full_step_bf16_vs_fp32_57600():
    from paper_2510_17519_b200.capi import Context
    from tests.gpu_common import nerr, to_cfg, to_samples
    cfg = O.paper_config(depth=1)
    gs = O.gate_std_for(cfg.hidden)
    P = O.open_gates(O.init_dit_params(cfg, O.Rng(1)), 2, gs, gs / 4)
    grid = O.Rng(3).uniform_tensor(GRID, -1.0, 1.0)
    text = O.Rng(4).normal_tensor((64, cfg.text_dim))
    s = O.make_batch([grid], 0.0, O.Rng(5))
    s[0].cond = True  # first-frame conditioning on
    out = {}
    for prec in ("fp32", "bf16"):
        ctx = Context(0, prec)
        ctx.upload(to_cfg(cfg), P)
        out[prec] = ctx.flow_step(to_samples(s), text, 8.0, grads=True, velocity=True)
        if prec == "bf16":  # bit-identical repeat
            again = ctx.flow_step(to_samples(s), text, 8.0, grads=False)
            assert again["loss"] == out[prec]["loss"] and again["grad_norm"] == out[prec]["grad_norm"]
        ctx.close()
    a, b = out["bf16"], out["fp32"]
    e_loss = abs(a["loss"] - b["loss"]) / abs(b["loss"])
    e_v = nerr(a["V"][0], b["V"][0])
    e_g = {k: nerr(a["grads"][k], b["grads"][k]) for k in b["grads"] if np.abs(b["grads"][k]).max() > 0}
    worst = max(e_g, key=e_g.get)
    print(f"57.6K step bf16 vs fp32: loss {e_loss:.2e} V {e_v:.2e} grad_norm "
          f"{abs(a['grad_norm'] - b['grad_norm']) / b['grad_norm']:.2e} worst grad {worst} {e_g[worst]:.2e}")
    assert np.isfinite(a["loss"]) and np.isfinite(b["loss"])
    assert e_loss <= 5e-2 and e_v <= 5e-2 and e_g[worst] <= 5e-2
