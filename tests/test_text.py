"""Text conditioning (dit.cpp:185-234): tokenize (host) and text_embed (device RMS-norm in the
reference's fp64 order) against the compiled reference, bit for bit."""
import ctypes

import numpy as np
import pytest

from oracle import oracle as O

needs_ref = pytest.mark.skipif(O.ref_lib() is None, reason="oracle/_ref not built (no reference sources)")
PROMPTS = ["a red cube sliding right", "", "   ", "two  clips\tand\nnewlines", "ünïcode wörds ✓ and ascii",
           " ".join(f"w{i}" for i in range(100))]


@needs_ref
@pytest.mark.parametrize("prompt", PROMPTS)
def test_tokenize_matches_reference(prompt):
    from paper_2510_17519_b200 import capi
    L = O.ref_lib()
    for vocab in (4096, 7, 1):
        n = L.ref_tokenize(prompt.encode(), vocab, None, 0)
        ref = np.empty(max(n, 1), dtype=np.int64)
        L.ref_tokenize(prompt.encode(), vocab, ref.ctypes.data, n)
        assert np.array_equal(capi.tokenize(prompt, vocab), ref[:n])


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("prompt,max_len", [(PROMPTS[0], 64), (PROMPTS[1], 64), (PROMPTS[5], 64), (PROMPTS[3], 2)])
def test_text_embed_bit_identical(prompt, max_len):
    from paper_2510_17519_b200 import capi
    from tests.golden.make_golden import CASES, build_case
    from tests.gpu_common import to_cfg
    cfg, P, _, _ = build_case("tiny", CASES["tiny"])
    r = O.Rng(4)
    vocab, D = 97, 48
    table, null = r.normal_tensor((vocab, D)), r.normal_tensor((1, D))
    ids = capi.tokenize(prompt, vocab)
    ctx = capi.Context(0, "fp32")
    ctx.upload(to_cfg(cfg), P)
    out, trunc = ctx.text_embed(ids, table, null, max_len)
    L = O.ref_lib()
    ref = np.empty((max(1, min(len(ids), max_len)), D))
    tr = ctypes.c_int()
    idsc = np.ascontiguousarray(ids, dtype=np.int64)
    n = L.ref_text_embed(idsc.ctypes.data if len(ids) else None, len(ids), table.ctypes.data, vocab, null.ctypes.data,
                         D, max_len, ref.ctypes.data, ctypes.byref(tr))
    assert n == out.shape[0] and trunc == bool(tr.value)
    assert out.tobytes() == ref.tobytes()
    with pytest.raises(capi.InputError):  # ids outside the vocabulary (dit.cpp:214-216)
        ctx.text_embed(np.array([vocab]), table, null, max_len)
    ctx.close()
