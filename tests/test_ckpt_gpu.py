"""Checkpoint -> device: mgv_params_upload_ckpt and mgv_params_save.

A checkpoint loaded into the device must give the same weights, and the same flow step bit-for-bit, as
uploading the same ParameterSet directly.  Saving the device parameters after AdamW steps must round-trip
bit-exactly (f32 payload = the fp32 masters) and load in the reference's own load_checkpoint."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.golden.make_golden import CASES, build_case
from tests.gpu_common import to_cfg, to_samples

pytestmark = pytest.mark.gpu


def _step(ctx, samples, text):
    return ctx.flow_step(to_samples(samples), text, 8.0, grads=True, velocity=True)


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
@pytest.mark.parametrize("f32_payload", [False, True])
def test_upload_from_checkpoint_matches_direct_upload(tmp_path, prec, f32_payload):
    from paper_2510_17519_b200 import capi
    cfg, P, text, samples = build_case("hd144", CASES["hd144"])
    extra = {"vae.enc.w": np.ones((2, 2)), "text.table": np.zeros(3)}  # non-dit.* entries are ignored
    path = tmp_path / "w.bin"
    dts = {k: capi.F32 if f32_payload else capi.F64 for k in list(P) + list(extra)}
    capi.save_checkpoint(path, {**P, **extra}, dtypes=dts, metadata={"stage": "pretrain"})
    ck = capi.load_checkpoint(path)
    direct = {k: (v.astype(np.float32).astype(np.float64) if f32_payload else v) for k, v in P.items()}
    a, b = capi.Context(0, prec), capi.Context(0, prec)
    a.upload(to_cfg(cfg), direct)
    b.upload_checkpoint(to_cfg(cfg), ck)
    assert a.names == b.names
    wa, wb = a.download(), b.download()
    for k in wa:
        assert wa[k].tobytes() == wb[k].tobytes(), k
    ra, rb = _step(a, samples, text), _step(b, samples, text)
    assert ra["loss"] == rb["loss"] and ra["grad_norm"] == rb["grad_norm"]
    for i in range(len(samples)):
        assert np.array_equal(ra["V"][i], rb["V"][i])
    for k in ra["grads"]:
        assert np.array_equal(ra["grads"][k], rb["grads"][k]), k
    a.close()
    b.close()


def test_checkpoint_missing_parameter_is_input_error(tmp_path):
    from paper_2510_17519_b200 import capi
    cfg, P, _, _ = build_case("tiny", CASES["tiny"])
    P = dict(P)
    P.pop("dit.out.b")
    capi.save_checkpoint(tmp_path / "m.bin", P)
    ctx = capi.Context(0, "fp32")
    with pytest.raises(capi.InputError):
        ctx.upload_checkpoint(to_cfg(cfg), capi.load_checkpoint(tmp_path / "m.bin"))
    ctx.close()


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_save_trained_parameters(tmp_path, dtype):
    from paper_2510_17519_b200 import capi
    cfg, P, text, samples = build_case("hd144", CASES["hd144"])
    ctx = capi.Context(0, "bf16")
    ctx.set_adamw(lr=1e-3, eps=1.0)
    ctx.upload(to_cfg(cfg), P)
    ctx.flow_step(to_samples(samples), text, 8.0)
    ctx.flow_step(to_samples(samples), text, 8.0)
    trained = ctx.download()
    path = tmp_path / "trained.bin"
    meta = {"step": "2", "stage": "sft"}
    ctx.save_checkpoint(path, dtype=capi.F32 if dtype == "f32" else capi.F64, metadata=meta)
    ck = capi.load_checkpoint(path)
    assert ck.metadata() == meta and ck.names() == sorted(trained)
    for k, v in trained.items():
        got = ck[k]
        assert got.shape == P[k].shape and got.ravel().tobytes() == v.tobytes(), k
        assert ck.dtype(k) == (capi.F32 if dtype == "f32" else capi.F64)
    # resume: a fresh context from the saved file continues from the same weights
    ctx2 = capi.Context(0, "bf16")
    ctx2.upload_checkpoint(to_cfg(cfg), ck)
    w2 = ctx2.download()
    for k in trained:
        assert w2[k].tobytes() == trained[k].tobytes(), k
    if O.ref_lib() is not None:  # the reference's loader reads the file identically
        st, vals, dts, rmeta = O.ref_ckpt_load(path)
        assert st == "ok" and rmeta == meta
        for k in trained:
            assert vals[k].ravel().tobytes() == trained[k].tobytes(), k
    ctx.close()
    ctx2.close()
