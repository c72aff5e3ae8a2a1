"""CPU checks of the C ABI boundary: the product library loads and exports every
symbol include/mugv_b200.h declares; without a GPU, context creation fails cleanly."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mugv_b200.h")


def header_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mgv_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = header_symbols()
    for s in ["mgv_ctx_create", "mgv_params_upload", "mgv_predict_velocity", "mgv_dit_forward", "mgv_flow_step",
              "mgv_flow_loss", "mgv_latent_rows", "mgv_rows_to_grid", "mgv_flow_step_device"]:
        assert s in syms, s


def test_library_exports_every_declared_symbol():
    from paper_2510_17519_b200._lib import lib
    L = lib()
    missing = [s for s in header_symbols() if not hasattr(L, s)]
    assert not missing, missing


def test_python_mirror_covers_exports():
    from paper_2510_17519_b200 import capi
    assert set(capi.EXPORTS) == set(header_symbols())


def test_no_gpu_context_fails_cleanly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2510_17519_b200.capi import Context, MugvError
    with pytest.raises(MugvError):
        Context(0, "bf16")


def test_library_is_sm100a_code():
    """The product .so carries sm_100a SASS with tcgen05 MMAs and TMA loads (no legacy HMMA path)."""
    import subprocess
    so = os.path.join(ROOT, "paper_2510_17519_b200", "libmugv_b200.so")
    out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", so], capture_output=True, text=True).stdout or \
        "arch = sm_100a" in out
    assert "UTCHMMA" in out and "UTMALDG" in out
    assert " HMMA" not in out
