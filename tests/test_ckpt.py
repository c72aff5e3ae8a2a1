"""MUGVCKPT container: the product's C++ reader/writer (mgv_ckpt_*) against the
reference's save_checkpoint / load_checkpoint (proj/src/params.cpp:92-225, compiled into oracle/_ref).

Mirrors the reference's own suite, proj/tests/test_formats.cpp:57-172 (round trip, f32 rounding, byte
stability, payload tiling, the CheckpointError taxonomy, the reserved name), and adds byte-for-byte and
cross-loading parity with the live reference plus header edge cases.  Host-only: runs without a GPU."""
import json
import os
import struct

import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_17519_b200 import capi

needs_ref = pytest.mark.skipif(O.ref_lib() is None, reason="oracle/_ref not built (no reference sources)")


def sample_params():
    """test_formats.cpp:44-53 (Rng(123) draws, two metadata strings)."""
    r = O.Rng(123)
    ps = {"alpha.w": r.normal_tensor((3, 4)), "beta.b": r.normal_tensor((5,)), "gamma": r.normal_tensor((2, 2, 2))}
    return ps, {"stage": "test", "step": "17"}


def craft(header: dict, payload: bytes) -> bytes:
    """test_formats.cpp:32-41; the header is dumped like nlohmann's dump() (compact, sorted keys)."""
    head = json.dumps(header, separators=(",", ":"), sort_keys=True, ensure_ascii=False).encode()
    return b"MUGVCKPT" + struct.pack("<Q", len(head)) + head + payload


def load_kind(path):
    try:
        capi.load_checkpoint(path)
    except capi.CheckpointError as e:
        return e.ckpt_kind
    return None


def test_round_trip_bit_exact(tmp_path):
    ps, meta = sample_params()
    p = tmp_path / "rt.bin"
    capi.save_checkpoint(p, ps, metadata=meta)
    ck = capi.load_checkpoint(p)
    assert ck.names() == sorted(ps)
    for k, v in ps.items():
        got = ck[k]
        assert got.shape == v.shape and got.tobytes() == v.tobytes()
        assert ck.dtype(k) == capi.F64
    assert ck.metadata() == meta


def test_f32_rounds_once_then_round_trips(tmp_path):
    w = O.Rng(7).normal_tensor((16,))
    a_path, b_path = tmp_path / "f32.bin", tmp_path / "f32b.bin"
    capi.save_checkpoint(a_path, {"w": w}, dtypes={"w": capi.F32})
    a = capi.load_checkpoint(a_path)
    assert np.array_equal(a["w"], w.astype(np.float32).astype(np.float64))
    capi.save_checkpoint(b_path, {"w": a["w"]}, dtypes={"w": capi.F32})
    b = capi.load_checkpoint(b_path)
    assert a["w"].tobytes() == b["w"].tobytes()
    assert a_path.read_bytes() == b_path.read_bytes()


def test_byte_stable_and_tiled(tmp_path):
    ps, meta = sample_params()
    capi.save_checkpoint(tmp_path / "s1.bin", ps, metadata=meta)
    capi.save_checkpoint(tmp_path / "s2.bin", dict(reversed(list(ps.items()))), metadata=meta)  # order-free
    raw = (tmp_path / "s1.bin").read_bytes()
    assert raw == (tmp_path / "s2.bin").read_bytes()
    hl = struct.unpack("<Q", raw[8:16])[0]
    header = json.loads(raw[16:16 + hl])
    ext = sorted((d["offset"], d["length"]) for k, d in header.items() if k != "__meta__")
    cursor = 0
    for off, ln in ext:
        assert off == cursor
        cursor = off + ln
    assert cursor == len(raw) - 16 - hl


@pytest.mark.parametrize("case", ["bad_magic", "short_payload", "short_header", "overlap", "gap", "not_json",
                                  "bad_length", "missing"])
def test_error_taxonomy(tmp_path, case):
    """test_formats.cpp:111-167, each subcase; the live reference must agree on the kind."""
    ps, meta = sample_params()
    good_path = tmp_path / "good.bin"
    capi.save_checkpoint(good_path, ps, metadata=meta)
    good = good_path.read_bytes()
    p = tmp_path / f"{case}.bin"
    expect = {"bad_magic": "BadMagic", "short_payload": "Truncated", "short_header": "Truncated",
              "overlap": "BadOffsets", "gap": "BadOffsets", "not_json": "BadHeader", "bad_length": "BadHeader",
              "missing": "Io"}[case]
    if case == "bad_magic":
        p.write_bytes(b"X" + good[1:])
    elif case == "short_payload":
        p.write_bytes(good[:-5])
    elif case == "short_header":
        p.write_bytes(good[:12])
    elif case == "overlap":
        h = {"a": {"dtype": "f64", "shape": [2], "offset": 0, "length": 16},
             "b": {"dtype": "f64", "shape": [2], "offset": 8, "length": 16}}
        p.write_bytes(craft(h, bytes(24)))
    elif case == "gap":
        h = {"a": {"dtype": "f64", "shape": [1], "offset": 0, "length": 8},
             "b": {"dtype": "f64", "shape": [1], "offset": 16, "length": 8}}
        p.write_bytes(craft(h, bytes(24)))
    elif case == "not_json":
        p.write_bytes(b"MUGVCKPT" + struct.pack("<Q", 3) + b"{{{")
    elif case == "bad_length":
        h = {"a": {"dtype": "f64", "shape": [2], "offset": 0, "length": 24}}
        p.write_bytes(craft(h, bytes(24)))
    assert load_kind(p) == expect
    if O.ref_lib() is not None:
        assert O.ref_ckpt_load(p) == ("error", expect)


def test_reserved_name_rejected(tmp_path):
    with pytest.raises(capi.InputError):
        capi.save_checkpoint(tmp_path / "r.bin", {"__meta__": np.array(1.0)})
    assert not (tmp_path / "r.bin").exists()


@needs_ref
@pytest.mark.parametrize("f32", [False, True])
def test_bytes_identical_to_reference_writer(tmp_path, f32):
    """Same ParameterSet -> the same file bytes as the reference's save_checkpoint, at the 10B-shaped block
    names (plus a scalar, an empty tensor and non-ASCII / escaped metadata)."""
    r = O.Rng(11)
    ps = {"dit.blk.0.attn.temp": r.normal_tensor((24,)), "dit.blk.0.attn.qkv.w": r.normal_tensor((12, 7)),
          "dit.patch.b": r.normal_tensor((9,)), "scalar": np.array(3.25), "empty": np.zeros((0, 3)),
          "Zeta": r.normal_tensor((2,)), "_under": r.normal_tensor((1,))}
    dts = {k: (0 if f32 and i % 2 == 0 else 1) for i, k in enumerate(ps)}
    meta = {"stage": "pre\"train\\\n\t", "ünï": "cødé ✓", "ctl": "\x01\x1f", "step": "17"}
    ours, ref = tmp_path / "ours.bin", tmp_path / "ref.bin"
    capi.save_checkpoint(ours, ps, dtypes=dts, metadata=meta)
    assert O.ref_ckpt_save(ref, ps, dtypes=dts, metadata=meta) == (0, None)
    assert ours.read_bytes() == ref.read_bytes()


@needs_ref
def test_cross_loading_with_reference(tmp_path):
    """A reference-written file loads identically in the product and vice versa (values, dtypes, metadata)."""
    r = O.Rng(5)
    ps = {f"t{i}": r.normal_tensor((i + 1, 3)) for i in range(5)}
    dts = {k: i % 2 for i, k in enumerate(ps)}
    meta = {"a": "1", "b": "two"}
    ref_file, our_file = tmp_path / "ref.bin", tmp_path / "ours.bin"
    O.ref_ckpt_save(ref_file, ps, dtypes=dts, metadata=meta)
    ck = capi.load_checkpoint(ref_file)
    st, vals, rdts, rmeta = O.ref_ckpt_load(ref_file)
    assert st == "ok" and ck.names() == sorted(vals) and ck.metadata() == rmeta == meta
    for k in vals:
        assert ck[k].tobytes() == vals[k].tobytes() and ck.dtype(k) == rdts[k]
    capi.save_checkpoint(our_file, ck.to_dict(), dtypes={k: ck.dtype(k) for k in ck.names()},
                         metadata=ck.metadata())
    assert our_file.read_bytes() == ref_file.read_bytes()


# header spellings the writer never produces; the product reader must decide each exactly as the reference
EDGE_HEADERS = {
    "whitespace": b' { "a" : { "dtype" : "f64" , "shape" : [ 1 ] , "offset" : 0 , "length" : 8 } } ',
    "escaped_name": b'{"\\u00e9\\"x":{"dtype":"f64","shape":[1],"offset":0,"length":8}}',
    "surrogate_pair": b'{"\\ud83d\\ude00":{"dtype":"f64","shape":[1],"offset":0,"length":8}}',
    "lone_surrogate": b'{"\\ud83d":{"dtype":"f64","shape":[1],"offset":0,"length":8}}',
    "bom": b'\xef\xbb\xbf{"a":{"dtype":"f64","shape":[1],"offset":0,"length":8}}',
    "duplicate_key": b'{"a":{"dtype":"f64","shape":[9],"offset":0,"length":72},'
                     b'"a":{"dtype":"f64","shape":[1],"offset":0,"length":8}}',
    "float_offset": b'{"a":{"dtype":"f64","shape":[1],"offset":0.0,"length":8}}',
    "float_shape": b'{"a":{"dtype":"f64","shape":[1.0],"offset":0,"length":8}}',
    "negative_shape": b'{"a":{"dtype":"f64","shape":[-1],"offset":0,"length":8}}',
    "scalar_shape": b'{"a":{"dtype":"f64","shape":1,"offset":0,"length":8}}',
    "null_shape": b'{"a":{"dtype":"f64","shape":null,"offset":0,"length":8}}',
    "unknown_dtype": b'{"a":{"dtype":"f16","shape":[1],"offset":0,"length":8}}',
    "incomplete": b'{"a":{"dtype":"f64","shape":[1],"offset":0}}',
    "meta_not_object": b'{"__meta__":[],"a":{"dtype":"f64","shape":[1],"offset":0,"length":8}}',
    "meta_not_string": b'{"__meta__":{"k":1},"a":{"dtype":"f64","shape":[1],"offset":0,"length":8}}',
    "header_array": b'[1,2]',
    "trailing_comma": b'{"a":{"dtype":"f64","shape":[1],"offset":0,"length":8},}',
    "trailing_garbage": b'{"a":{"dtype":"f64","shape":[1],"offset":0,"length":8}} x',
    "leading_zero": b'{"a":{"dtype":"f64","shape":[01],"offset":0,"length":8}}',
    "raw_control": b'{"a\x01":{"dtype":"f64","shape":[1],"offset":0,"length":8}}',
    "bad_utf8": b'{"a\xc3\x28":{"dtype":"f64","shape":[1],"offset":0,"length":8}}',
    "past_end": b'{"a":{"dtype":"f64","shape":[1],"offset":8,"length":8}}',
    "trailing_payload": b'{"a":{"dtype":"f64","shape":[],"offset":0,"length":8}}',
    "zero_len_between": b'{"a":{"dtype":"f64","shape":[0],"offset":8,"length":0},'
                        b'"b":{"dtype":"f64","shape":[1],"offset":0,"length":8}}',
    "sorted_error_order": b'{"a":{"dtype":"f64","shape":[1],"offset":64,"length":8},'
                          b'"b":{"dtype":"f99","shape":[1],"offset":0,"length":8}}',
}


@needs_ref
@pytest.mark.parametrize("case", sorted(EDGE_HEADERS))
def test_header_edge_cases_match_reference(tmp_path, case):
    head = EDGE_HEADERS[case]
    payload = struct.pack("<d", 1.5) + (b"\0" * 8 if case == "trailing_payload" else b"")
    p = tmp_path / f"{case}.bin"
    p.write_bytes(b"MUGVCKPT" + struct.pack("<Q", len(head)) + head + payload)
    ref = O.ref_ckpt_load(p)
    if ref[0] == "error":
        assert ref[1] in O.REF_CKPT_KINDS.values(), ref  # cases chosen so the reference raises CheckpointError
        assert load_kind(p) == ref[1]
    else:
        ck = capi.load_checkpoint(p)
        _, vals, dts, meta = ref
        assert ck.names() == sorted(vals) and ck.metadata() == meta
        for k in vals:
            assert ck[k].shape == vals[k].shape and ck[k].tobytes() == vals[k].tobytes()
