"""Post-training losses on the hot-path forward (proj/src/posttrain.cpp).

CPU: the oracle's restatement (oracle.post_loss over flow_fwdbwd) is pinned to the live reference's
post_loss_graph + backward (oracle/_ref), and the product's scalar helpers / config validation are checked.
GPU (-m gpu): the product's device path -- mgv_flow_errors, mgv_flow_step_weighted, mgv_post_train_step,
mgv_post_pref_loss -- against the pinned oracle: fp32 mode <= 1e-4, bf16 mode <= 5e-2 (normwise)."""
import math

import numpy as np
import pytest

from oracle import oracle as O

needs_ref = pytest.mark.skipif(O.ref_lib() is None, reason="oracle/_ref not built (no reference sources)")

HP = dict(beta=1.5, alpha=0.7, w_d=1.2, w_u=0.8)


def tiny_cfg():
    """head_dim 144 with the paper rope split (the 10B head shape), 2 heads, depth 1."""
    return O.DitConfig(depth=1, hidden=288, heads=2, text_dim=64, c_z=24, rope_split=(48, 48, 48))


GS = O.gate_std_for(288) * 4  # gate scale of the hd144 golden case


def records(cfg, tag):
    """Records on two grids (first-frame masked U=2 clip, unmasked U=1 image), per-record texts and fps."""
    r = O.Rng(31)
    texts = [r.normal_tensor((5, cfg.text_dim)), r.normal_tensor((3, cfg.text_dim))]

    def rec(grid_shape, cond, ti, fps):
        rows, coords, dims = O.latent_rows(r.uniform_tensor(grid_shape, -1.0, 1.0))
        return O.Record(dims, rows, cond, texts[ti], fps, coords)

    if tag == "dpo":  # (winner, loser) pairs share grid, mask and text
        return [rec((2, 4, 8, 24), True, 0, 8.0), rec((2, 4, 8, 24), True, 0, 8.0),
                rec((1, 4, 6, 24), False, 1, 12.0), rec((1, 4, 6, 24), False, 1, 12.0)], None
    return [rec((2, 4, 8, 24), True, 0, 8.0), rec((1, 4, 6, 24), False, 1, 12.0),
            rec((2, 2, 4, 24), False, 0, 6.0)], [1, 0, 1]


def sft_batch(cfg):
    r = O.Rng(41)
    grids = [r.uniform_tensor((2, 4, 4, 24), -1.0, 1.0), r.uniform_tensor((1, 2, 4, 24), -1.0, 1.0)]
    s = O.make_batch(grids, 0.0, O.Rng(42))
    s[0].cond = True
    return s, r.normal_tensor((4, cfg.text_dim)), 8.0


def models(cfg):
    """policy and frozen reference: same init, different gate draws (so the DPO/KTO margins are non-zero)."""
    pol = O.RefModel(cfg, 1, 2, GS, GS / 4)
    ref = O.RefModel(cfg, 1, 9, GS, GS / 4)
    return pol, ref


def shaped(P, like):
    return {k: P[k].reshape(like[k].shape) for k in P}


@needs_ref
@pytest.mark.parametrize("tag", ["dpo", "kto"])
def test_post_loss_restatement_matches_reference(tag):
    cfg = tiny_cfg()
    pol, ref = models(cfg)
    init = O.init_dit_params(cfg, O.Rng(1))
    Ppol, Pref = shaped(pol.params(), init), shaped(ref.params(), init)
    recs, des = records(cfg, tag)
    sft, stx, sfps = sft_batch(cfg)
    o = O.post_loss(Ppol, Pref, cfg, tag, recs, des, sft, stx, sfps, seed=77, **HP)
    r = O.ref_post_loss(pol.h, ref.h, cfg, tag, recs, des, sft, stx, sfps, 77, **HP, names=pol.names,
                        numels=[Ppol[k].size for k in pol.names])
    for key in ("total", "preference", "sft", "grad_norm"):
        assert abs(o[key] - r[key]) <= 1e-12 * max(1.0, abs(r[key])), (key, o[key], r[key])
    assert abs(o["preference"]) > 1e-3  # a non-degenerate margin
    for k in pol.names:
        g, gr = o["grads"][k].ravel(), r["grads"][k]
        den = max(np.abs(gr).max(), 1e-300)
        assert np.abs(g - gr).max() <= 1e-10 * den or np.abs(gr).max() == 0, k


def test_scalar_helpers():
    from paper_2510_17519_b200 import capi
    # dpo_from_errors = softplus(-beta((e_ref_w - e_th_w) - (e_ref_l - e_th_l)))   posttrain.cpp:144-147
    m = 1.3 * ((0.4 - 0.5) - (0.9 - 0.2))
    assert capi.dpo_from_errors(0.5, 0.2, 0.4, 0.9, 1.3) == pytest.approx(math.log1p(math.exp(-m)), rel=1e-15)
    # DPO at theta = ref is log 2 (test_posttrain.cpp:176-233)
    assert capi.dpo_from_errors(0.3, 0.7, 0.3, 0.7, 2.0) == pytest.approx(math.log(2.0), rel=1e-15)
    rw, des = [0.1, 0.4, -0.2, 0.0], [1, 0, 1, 0]
    z0 = sum(rw) / 4
    sig = lambda x: 1.0 / (1.0 + math.exp(-x))  # noqa: E731
    want = sum(1.2 * (1 - sig(r - z0)) if d else 0.8 * (1 - sig(z0 - r)) for r, d in zip(rw, des)) / 4
    assert capi.kto_from_rewards(rw, des, 1.2, 0.8) == pytest.approx(want, rel=1e-14)
    # KTO at identical rewards = w/2 (test_posttrain.cpp:264-312)
    assert capi.kto_from_rewards([0.3, 0.3], [1, 1], 1.0, 1.0) == pytest.approx(0.5, rel=1e-15)
    assert capi.kto_from_rewards([0.5], [1], 1.0, 1.0, z0=0.5) == pytest.approx(0.5, rel=1e-15)


@pytest.mark.parametrize("field,value,msg", [("beta", 0.0, "beta must be > 0"),
                                             ("alpha_sft", -1.0, "alpha_sft must be >= 0"),
                                             ("gamma_merge", 1.5, "gamma_merge must lie in (0, 1]"),
                                             ("w_u", 0.0, "kto weights must be > 0"),
                                             ("interleave", (), "interleave plan must not be empty"),
                                             ("interleave", ("dpo", "sft"), "unknown interleave tag: sft")])
def test_config_validation(field, value, msg):
    import ctypes
    from paper_2510_17519_b200 import capi
    cfg = capi.PostTrainConfig()
    setattr(cfg, field, value)
    c = cfg.to_c()
    buf = ctypes.create_string_buffer(256)
    st = capi._lib().mgv_post_validate(ctypes.byref(c), buf, 256)
    assert st == 2 and buf.value.decode() == msg  # ConfigError with the reference's message (posttrain.cpp:37-49)
    assert capi._lib().mgv_post_validate(ctypes.byref(capi.PostTrainConfig().to_c()), buf, 256) == 0


# ------------------------------------------------------------------------------------------------ GPU
def _product_records(recs, capi):
    return [capi.SampleRecord(r.dims, r.coords, r.rows, r.text, r.fps,
                              (r.coords[:, 0] == 0).astype(np.uint8) if r.cond else None) for r in recs]


def _ctx(cfg, P, prec, capi):
    from tests.gpu_common import to_cfg
    c = capi.Context(0, prec)
    c.upload(to_cfg(cfg), P)
    return c


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_weighted_step_gradients(prec):
    """mgv_flow_step_weighted: per-record text / fps, signed weights -> sum_k w_k dl_k vs the oracle."""
    from paper_2510_17519_b200 import capi
    from tests.gpu_common import nerr, to_samples
    cfg = tiny_cfg()
    P = O.open_gates(O.init_dit_params(cfg, O.Rng(1)), 2, GS, GS / 4)
    recs, _ = records(cfg, "kto")
    rng = O.Rng(5)
    draws = [O.make_draw(r, rng) for r in recs]
    weights = [0.7, -0.3, 1.1]
    samples = [O.Sample(r.dims, r.rows, d[1], d[0], r.cond, r.coords) for r, d in zip(recs, draws)]
    G = {k: np.zeros_like(v) for k, v in P.items()}
    errs = []
    for s, r, w in zip(samples, recs, weights):
        o = O.flow_fwdbwd(P, cfg, [s], r.text, r.fps, grads=True)
        errs.append(o["loss"])
        for k in G:
            G[k] += w * o["grads"][k]
    ctx = _ctx(cfg, P, prec, capi)
    ev = [(fs, r.text, r.fps) for fs, r in zip(to_samples(samples), recs)]
    e_fwd = ctx.flow_errors(ev)
    out = ctx.flow_step_weighted(ev, weights, grads=True)
    tol = 1e-4 if prec == "fp32" else 5e-2
    assert np.array_equal(e_fwd, out["errs"])  # the forward-only pass and the step see the same errors
    assert nerr(out["errs"], errs) <= tol
    assert abs(out["loss"] - sum(w * e for w, e in zip(weights, errs))) <= tol * sum(abs(e) for e in errs)
    worst = max(nerr(out["grads"][k], G[k]) for k in G if np.abs(G[k]).max() > 0)
    assert worst <= tol, worst
    assert out["grad_norm"] == pytest.approx(O.grad_norm(G), rel=tol)
    ctx.close()


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("tag", ["dpo", "kto"])
def test_post_train_step_matches_oracle(prec, tag):
    """post_train_step on device: metrics vs the oracle, then the AdamW update (eps = 1, smooth) of the
    policy weights vs the oracle's AdamW applied to the oracle's post-training gradients."""
    from paper_2510_17519_b200 import capi
    cfg = tiny_cfg()
    init = O.init_dit_params(cfg, O.Rng(1))
    Ppol = O.open_gates({k: v.copy() for k, v in init.items()}, 2, GS, GS / 4)
    Pref = O.open_gates({k: v.copy() for k, v in init.items()}, 9, GS, GS / 4)
    recs, des = records(cfg, tag)
    sft, stx, sfps = sft_batch(cfg)
    seed = 123
    o = O.post_loss(Ppol, Pref, cfg, tag, recs, des, sft, stx, sfps, seed=seed, **HP)
    pol, ref = _ctx(cfg, Ppol, prec, capi), _ctx(cfg, Pref, prec, capi)
    st = capi.PostTrainState(pol, ref, lr=1e-3, seed=seed)
    pol.set_adamw(lr=1e-3, eps=1.0)  # smooth AdamW direction for the comparison
    pcfg = capi.PostTrainConfig(beta=HP["beta"], alpha_sft=HP["alpha"], w_d=HP["w_d"], w_u=HP["w_u"],
                                interleave=(tag,))
    prs = _product_records(recs, capi)
    from tests.gpu_common import to_samples
    if tag == "dpo":
        m = st.train_step(pcfg, "dpo", pairs=[(prs[0], prs[1]), (prs[2], prs[3])], sft=to_samples(sft),
                          sft_text=stx, sft_fps=sfps)
    else:
        m = st.train_step(pcfg, "kto", labels=list(zip(prs, des)), sft=to_samples(sft), sft_text=stx, sft_fps=sfps)
    tol = 1e-4 if prec == "fp32" else 5e-2
    print(prec, tag, m, {k: o[k] for k in ("total", "preference", "sft", "grad_norm")})
    for key in ("total", "preference", "sft", "grad_norm"):
        assert abs(m[key] - o[key]) <= tol * max(1.0, abs(o[key])), (key, m[key], o[key])
    assert st.plan_pos == 1
    got = pol.download()
    refw = {k: v.copy() for k, v in Ppol.items()}
    opt = O.AdamW(1e-3, 0.9, 0.999, 1.0, 0.0)
    opt.update(refw, o["grads"])
    errs = {}
    for k in refw:
        upd = refw[k].ravel() - Ppol[k].ravel()
        if np.abs(upd).max() == 0:
            continue
        excess = np.abs(got[k] - refw[k].ravel()) - 4 * 2.0 ** -24 * np.abs(refw[k].ravel())
        errs[k] = max(float(excess.max()), 0.0) / float(np.abs(upd).max())
    worst = max(errs, key=errs.get)
    assert errs[worst] <= tol, (worst, errs[worst])
    # the frozen reference is untouched
    wr = ref.download()
    for k in Pref:
        assert np.array_equal(wr[k], Pref[k].astype(np.float32).astype(np.float64).ravel()), k
    st.close()
    pol.close()
    ref.close()


@pytest.mark.gpu
def test_post_schedule_and_pref_loss():
    from paper_2510_17519_b200 import capi
    from tests.gpu_common import to_samples
    cfg = tiny_cfg()
    init = O.init_dit_params(cfg, O.Rng(1))
    Ppol = O.open_gates({k: v.copy() for k, v in init.items()}, 2, GS, GS / 4)
    Pref = O.open_gates({k: v.copy() for k, v in init.items()}, 9, GS, GS / 4)
    pol, ref = _ctx(cfg, Ppol, "fp32", capi), _ctx(cfg, Pref, "fp32", capi)
    recs, des = records(cfg, "kto")
    prs = _product_records(recs, capi)
    pcfg = capi.PostTrainConfig(beta=HP["beta"], alpha_sft=HP["alpha"], w_d=HP["w_d"], w_u=HP["w_u"])
    # dpo_loss / kto_loss values (forward only) vs the oracle's preference term
    for tag, kw, orecs, odes in [("kto", dict(labels=list(zip(prs, des))), recs, des)]:
        v = capi.post_pref_loss(pol, ref, pcfg, tag, seed=9, **kw)
        sft, stx, sfps = sft_batch(cfg)
        o = O.post_loss(Ppol, Pref, cfg, tag, orecs, odes, sft, stx, sfps, seed=9, grads=False, **HP)
        assert abs(v - o["preference"]) <= 1e-4 * max(1.0, abs(o["preference"]))
    # the interleave plan ("dpo", "kto"): a kto batch first is a SchedulingError and leaves the plan alone
    st = capi.PostTrainState(pol, ref, lr=1e-4, seed=1)
    sft, stx, sfps = sft_batch(cfg)
    with pytest.raises(capi.SchedulingError):
        st.train_step(pcfg, "kto", labels=list(zip(prs, des)), sft=to_samples(sft), sft_text=stx, sft_fps=sfps)
    assert st.plan_pos == 0
    with pytest.raises(capi.InputError):  # empty SFT batch (posttrain.cpp:275)
        st.train_step(pcfg, "dpo", pairs=[(prs[0], prs[0])], sft=[], sft_text=stx)
    assert st.plan_pos == 0
    st.close()
    pol.close()
    ref.close()


@needs_ref
def test_merge_weights_and_anneal_lr_match_reference():
    import ctypes
    from paper_2510_17519_b200 import capi
    L = O.ref_lib()
    for k, gamma in [(1, 0.9), (4, 0.9), (7, 0.5), (3, 1.0)]:
        ref = np.empty(k)
        assert L.ref_merge_weights(k, gamma, ref.ctypes.data) == 0
        assert capi.merge_weights(k, gamma).tobytes() == ref.tobytes()
    for step, a, b, n in [(0, 1e-4, 1e-6, 1000), (1, 1e-4, 1e-6, 1000), (500, 1e-4, 1e-6, 1000), (999, 1e-4, 1e-6, 1000),
                          (5000, 3e-4, 0.0, 10), (1, 1.0, 1.0, 2)]:
        ref = ctypes.c_double()
        assert L.ref_anneal_lr(step, a, b, n, ctypes.byref(ref)) == 0
        assert capi.anneal_lr(step, a, b, n) == ref.value
    with pytest.raises(capi.ConfigError):
        capi.merge_weights(3, 1.5)
    with pytest.raises(capi.ConfigError):
        capi.anneal_lr(0, 1e-6, 1e-4, 10)


@pytest.mark.gpu
@needs_ref
def test_rdpo_pairs_match_reference():
    """rdpo_pairs (posttrain.cpp:235-254) on the device sampler (fp32 mode) against the reference."""
    import ctypes
    from paper_2510_17519_b200 import capi
    from tests.gpu_common import nerr
    cfg = tiny_cfg()
    pol, _ = models(cfg)
    init = O.init_dit_params(cfg, O.Rng(1))
    P = shaped(pol.params(), init)
    recs, _ = records(cfg, "kto")
    ctx = _ctx(cfg, P, "fp32", capi)
    got = capi.rdpo_pairs(ctx, _product_records(recs, capi), steps=3, seed=77)
    RR = type("RefRecord", (ctypes.Structure,), {"_fields_": [
        ("dims", ctypes.c_int64 * 3), ("rows", ctypes.c_void_p), ("cond", ctypes.c_int32), ("text", ctypes.c_void_p),
        ("L", ctypes.c_int64), ("fps", ctypes.c_double)]})
    arr = (RR * len(recs))()
    keep = []
    for i, r in enumerate(recs):
        rows, tx = np.ascontiguousarray(r.rows), np.ascontiguousarray(r.text)
        keep += [rows, tx]
        arr[i].dims[:] = list(r.dims)
        arr[i].rows, arr[i].cond, arr[i].text, arr[i].L, arr[i].fps = rows.ctypes.data, int(r.cond), \
            tx.ctypes.data, tx.shape[0], r.fps
    W = [np.empty_like(r.rows) for r in recs]
    Lo = [np.empty_like(r.rows) for r in recs]
    wp = (ctypes.c_void_p * len(recs))(*[w.ctypes.data for w in W])
    lp = (ctypes.c_void_p * len(recs))(*[x.ctypes.data for x in Lo])
    c = O.ref_cfg(cfg)
    assert O.ref_lib().ref_rdpo_pairs(pol.h, ctypes.addressof(c), len(recs), ctypes.addressof(arr), 3, 77, wp, lp) == 0
    for i in range(len(recs)):
        ew, el = nerr(got[i][0], W[i]), nerr(got[i][1], Lo[i])
        print(f"record {i}: winner {ew:.2e} loser {el:.2e}")
        assert ew < 1e-4 and el < 1e-4
    ctx.close()
