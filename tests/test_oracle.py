"""Pin the oracle (numpy/C restatement) against the reference: golden fixtures
generated from the reference itself (tests/golden/make_golden.py) and, when the
compiled reference (oracle/_ref) is present, live calls into it."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.golden.make_golden import ALL_CASES, CASES, LONG_CASES, build_case

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
needs_ref = pytest.mark.skipif(O.ref_lib() is None, reason="oracle/_ref not built (no reference sources)")


def nerr(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def check_against_golden(out, g, samples, tol=1e-12):
    """Compare a flow_fwdbwd result (V, loss, grads; taps optional) with a fixture the REFERENCE produced.
    Returns the worst normwise error per quantity (max |a-b| over the stored entries / max |ref|)."""
    errs = {"loss": abs(out["loss"] - float(g["loss"])) / abs(float(g["loss"]))}
    for i, s in enumerate(samples):
        assert bool(g[f"cond.{i}"]) == s.cond
        V = np.asarray(out["V"][i], dtype=np.float64).ravel()
        if f"V.{i}" in g:
            errs[f"V{i}"] = nerr(V, g[f"V.{i}"])
        else:
            vi = g[f"Vi.{i}"]
            errs[f"V{i}"] = float(np.abs(V[vi] - g[f"Vv.{i}"]).max() / float(g[f"Vmax.{i}"]))
            errs[f"|V{i}|"] = abs(np.linalg.norm(V) - float(g[f"Vn.{i}"])) / float(g[f"Vn.{i}"])
        if "taps" in out:
            taps = np.concatenate([t.ravel() for t in out["taps"][i]])
            assert nerr(taps[g[f"taps_idx.{i}"]], g[f"taps_val.{i}"]) < tol
            assert abs(np.linalg.norm(taps) - float(g[f"taps_norm.{i}"])) < tol * float(g[f"taps_norm.{i}"])
    for k, gv in out["grads"].items():
        gv = np.asarray(gv, dtype=np.float64).ravel()
        if f"g:{k}" in g:
            errs[k] = nerr(gv, g[f"g:{k}"])
            continue
        ref_n = float(g[f"gn:{k}"])
        if ref_n == 0.0:
            errs[k] = float(np.abs(gv).max())
            continue
        den = float(g[f"gm:{k}"]) if f"gm:{k}" in g else float(np.abs(g[f"gv:{k}"]).max())
        errs[k] = max(float(np.abs(gv[g[f"gi:{k}"]] - g[f"gv:{k}"]).max()) / den,
                      abs(np.linalg.norm(gv) - ref_n) / ref_n)
    return errs


@pytest.mark.parametrize("name", sorted(ALL_CASES))
def test_restatement_matches_golden(name):
    path = os.path.join(GOLDEN, f"{name}.npz")
    if name in LONG_CASES and not os.path.exists(path):
        pytest.skip("fixture not generated (tests/golden/make_golden.py " + name + ")")
    g = np.load(path)
    spec = json.loads(str(g["spec"]))
    cfg, P, text, samples = build_case(name, ALL_CASES[name])
    assert spec["cfg"]["hidden"] == cfg.hidden
    out = O.flow_fwdbwd(P, cfg, samples, text, 8.0, grads=True, with_taps=True)
    errs = check_against_golden(out, g, samples)
    worst = max(errs, key=errs.get)
    assert errs[worst] < 1e-11, (worst, errs[worst])


def test_flow_loss_hand_case():
    """proj/tests/test_flow.cpp:63-99: flow_loss = 5/3; masked rows get exactly zero gradient."""
    cfg = O.DitConfig(depth=1, hidden=12, heads=2, text_dim=6, c_z=2, rope_split=(2, 2, 2))
    pred = np.array([[1.0, 2.0, 3.0]])
    tgt = np.array([[0.0, 2.0, 5.0]])
    assert abs(float(np.mean((pred - tgt) ** 2)) - 5.0 / 3.0) < 1e-15
    # all-masked sample: U=1 with first-frame conditioning -> loss 0 and zero grads (SURVEY 8c side finding)
    P = O.open_gates(O.init_dit_params(cfg, O.Rng(1)), 2)
    g = O.Rng(3).uniform_tensor((1, 4, 4, 2), -1, 1)
    s = O.make_batch([g], 1.0, O.Rng(5))
    assert s[0].cond
    out = O.flow_fwdbwd(P, cfg, s, O.Rng(4).normal_tensor((2, 6)))
    assert out["loss"] == 0.0
    assert all(np.all(v == 0) for v in out["grads"].values())


def test_patch_rows_golden_positions():
    """proj/tests/test_dit.cpp:74-97 (bit-exact index math) via the C restatement."""
    grid = O.Rng(11).uniform_tensor((2, 8, 8, 24), -1.0, 1.0)
    rows, coords, dims = O.latent_rows(grid)
    assert rows.shape == (32, 96) and dims == (2, 4, 4)
    assert list(coords[0]) == [0, 0, 0] and list(coords[1]) == [0, 0, 1]
    assert list(coords[5]) == [0, 1, 1] and list(coords[16]) == [1, 0, 0]
    assert rows[1, 0] == grid[0, 0, 2, 0] and rows[1, 24] == grid[0, 0, 3, 0]
    assert np.array_equal(O.rows_to_grid(rows, coords, dims), grid)
    perm = np.random.default_rng(0).permutation(32)
    assert np.array_equal(O.rows_to_grid(rows[perm], coords[perm], dims), grid)
    bad = coords.copy()
    bad[3] = bad[4]
    with pytest.raises(ValueError):
        O.rows_to_grid(rows, bad, dims)


def test_default_rope_split():
    """dit.cpp:65-90; default_rope_split(64,{4,4,4}) = (22,22,20)."""
    assert O.default_rope_split(64, (4, 4, 4)) == (22, 22, 20)
    assert sum(O.default_rope_split(144, (16, 45, 80))) == 144


@needs_ref
def test_rng_matches_reference():
    L = O.ref_lib()
    for seed, skip, n, std in [(0, 0, 10, 1.0), (7, 3, 1001, 0.5), (2**63 + 5, 1, 4, 2.0)]:
        a = np.empty(n)
        L.ref_rng_normal_fill(seed, skip, n, std, a.ctypes.data)
        r = O.Rng(seed)
        for _ in range(skip):
            r.uniform()
        assert np.array_equal(a, r.normal_tensor((n,), std))
    a = np.empty(777)
    L.ref_rng_uniform_fill(99, 777, -1.0, 1.0, a.ctypes.data)
    assert np.array_equal(a, O.Rng(99).uniform_tensor((777,), -1.0, 1.0))


@needs_ref
def test_make_batch_matches_reference():
    import ctypes
    L = O.ref_lib()
    g = O.Rng(3)
    grids = [g.uniform_tensor(s, -1, 1) for s in [(2, 4, 4, 2), (3, 2, 6, 2), (1, 2, 2, 2)]]
    dims = np.array([x.shape[:3] for x in grids], dtype=np.int64)
    noise = [np.empty((x.shape[0] * x.shape[1] * x.shape[2] // 4, 8)) for x in grids]
    t = np.empty(3)
    m = np.empty(3, dtype=np.int32)
    gp = (ctypes.c_void_p * 3)(*[x.ctypes.data for x in grids])
    npp = (ctypes.c_void_p * 3)(*[x.ctypes.data for x in noise])
    assert L.ref_make_batch(3, dims.ctypes.data, 2, gp, 8.0, 0.5, 5, npp, t.ctypes.data, m.ctypes.data) == 0
    s = O.make_batch(grids, 0.5, O.Rng(5))
    for i in range(3):
        assert np.array_equal(s[i].noise, noise[i])
        assert s[i].t == t[i] and int(s[i].cond) == m[i]


@needs_ref
def test_restatement_matches_live_reference_10b_width():
    """10B dims (H3456, 24x144, text 64x4096), depth 1, N=8: fwd+bwd vs the reference."""
    cfg = O.paper_config(depth=1)
    gs = O.gate_std_for(cfg.hidden)
    ref = O.RefModel(cfg, 1, 2, gs, gs / 4)
    init = O.open_gates(O.init_dit_params(cfg, O.Rng(1)), 2, gs, gs / 4)
    grid = O.Rng(3).uniform_tensor((2, 2, 4, 24), -1.0, 1.0)
    text = O.Rng(4).normal_tensor((64, 4096))
    s = O.make_batch([grid], 0.0, O.Rng(5))
    s[0].cond = True
    r = ref.flow_fwdbwd(s, text, 8.0, grads=True)
    o = O.flow_fwdbwd(init, cfg, s, text, 8.0, grads=True)
    assert abs(r["loss"] - o["loss"]) < 1e-12 * abs(r["loss"])
    assert nerr(o["V"][0], r["V"][0]) < 1e-12
    for k in init:
        assert nerr(o["grads"][k], r["grads"][k]) < 1e-10 or np.abs(r["grads"][k]).max() == 0, k


def test_adamw_restatement_matches_reference():
    """oracle.AdamW (optim.cpp:7-24 restated) vs the reference's own AdamW::update, three steps."""
    ref_lib_available = os.path.exists(os.path.join(os.path.dirname(O.__file__), "_ref", "libmugv_ref.so"))
    if not ref_lib_available:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(3)
    P = {"dit.a": rng.standard_normal((4, 5)), "dit.b": rng.standard_normal(7)}
    Q = {k: v.copy() for k, v in P.items()}
    mine, theirs = O.AdamW(1e-2, 0.8, 0.95, 1e-6, 0.1), O.RefAdamW(1e-2, 0.8, 0.95, 1e-6, 0.1)
    for step in range(3):
        G = {k: rng.standard_normal(v.shape) for k, v in P.items()}
        mine.update(P, G)
        theirs.update(Q, G)
        for k in P:
            assert np.allclose(P[k], Q[k], rtol=0, atol=1e-14), (step, k)


@pytest.mark.parametrize("direction,cond", [(-1, False), (-1, True), (1, True)])
def test_sampler_restatement_matches_reference(direction, cond):
    """oracle.sample_rows (flowtrain.cpp:135-172 restated) vs the reference's forward/reverse_sample_rows."""
    if not os.path.exists(os.path.join(os.path.dirname(O.__file__), "_ref", "libmugv_ref.so")):
        pytest.skip("oracle/_ref not built")
    cfg = O.DitConfig(depth=1, hidden=24, heads=2, text_dim=6, c_z=2, rope_split=(4, 4, 4))
    ref = O.RefModel(cfg, 1, 2, 0.2, 0.05)
    P = O.open_gates(O.init_dit_params(cfg, O.Rng(1)), 2, 0.2, 0.05)  # bit-equal to ref's (test above)
    dims = (2, 2, 3)
    coords = O.grid_coords(dims)
    N, D = coords.shape[0], 4 * cfg.c_z
    x0 = O.Rng(7).normal_tensor((N, D))
    text = O.Rng(4).normal_tensor((3, 6))
    cm = (coords[:, 0] == 0).astype(np.uint8) if cond else None
    cl = O.Rng(8).normal_tensor((N, D)) if cond else None
    mine = O.sample_rows(P, cfg, x0, coords, text, 8.0, 3, direction, cm, cl)
    theirs = O.ref_sample_rows(ref, dims, x0, text, 8.0, 3, direction, cm, cl)
    assert np.abs(mine - theirs).max() <= 1e-12 * max(1.0, np.abs(theirs).max())


@needs_ref
def test_ref_rope3d_matches_restatement():
    """The reference veneer's Tape::rope3d (forward and the backward's inverse rotation) against the numpy
    restatement rope_tables / rope_apply (autodiff.cpp:851-898): equal up to libm / numpy trig rounding."""
    import ctypes
    L = O.ref_lib()
    rng = np.random.default_rng(5)
    split, heads, N = (22, 22, 20), 4, 50
    x = rng.standard_normal((N, heads * sum(split)))
    co = rng.integers(0, 50, size=(N, 3)).astype(np.int32)
    cos, sin = O.rope_tables(co, split)
    for inverse, direction in ((0, 1), (1, -1)):
        ref = np.empty_like(x)
        assert L.ref_rope3d(x.ctypes.data, N, heads, (ctypes.c_int * 3)(*split), co.ctypes.data, 10000.0, inverse,
                            ref.ctypes.data) == 0
        assert np.max(np.abs(ref - O.rope_apply(x, cos, sin, heads, direction))) < 1e-13


def mask_case(kind):
    """A U=3 sample of the hd144 config with a general unit-aligned ConditionMask (flowtrain.cpp:61-100) and
    condition latents different from the clean rows."""
    cfg, P, text, samples = build_case("hd144", CASES["hd144"])
    s = samples[1]  # dims (3, 1, 2): 3 latent units
    units = s.coords[:, 0]
    m = {"last": units == 2, "two": (units == 0) | (units == 2), "none": np.zeros_like(units, dtype=bool)}[kind]
    s.cond = False
    s.mask = m.astype(np.uint8)
    s.cond_latents = O.Rng(8).normal_tensor(s.clean.shape)
    return cfg, P, text, samples


@needs_ref
@pytest.mark.parametrize("kind", ["last", "two"])
def test_general_condition_mask_matches_reference(kind):
    """oracle.masked_input with an explicit unit-aligned mask and condition latents vs the reference's
    validate_mask + apply_condition_mask (flowtrain.cpp:61-100) inside FlowTrainer::step's fwd+bwd."""
    cfg, P, text, samples = mask_case(kind)
    gs = CASES["hd144"]["gate_std"]
    ref = O.RefModel(cfg, 1, 2, gs, gs / 4)
    r = ref.flow_fwdbwd(samples, text, 8.0, grads=True)
    o = O.flow_fwdbwd(P, cfg, samples, text, 8.0, grads=True)
    assert abs(r["loss"] - o["loss"]) <= 1e-12 * abs(r["loss"])
    for i in range(len(samples)):
        assert nerr(o["V"][i], r["V"][i]) < 1e-12
    for k in P:
        assert nerr(o["grads"][k], r["grads"][k]) < 1e-11 or np.abs(r["grads"][k]).max() == 0, k


def test_mask_must_cover_whole_units():
    cfg, P, text, samples = mask_case("last")
    samples[1].mask = samples[1].mask.copy()
    samples[1].mask[np.argmax(samples[1].coords[:, 0] == 2)] = 0  # one token of unit 2 unconditioned
    with pytest.raises(ValueError):
        O.masked_input(samples[1])
