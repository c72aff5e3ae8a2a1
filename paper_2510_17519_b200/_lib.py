"""Loader for the product library ``libmugv_b200.so`` (C++ runtime + sm_100a kernels).

There is no fallback: if the library is missing or fails to load, import
raises.  Build it with ``__graft_entry__.build()`` (or ``make -C
paper_2510_17519_b200/csrc``).
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# MGV_LIB_PATH lets the A/B tools in tools/ load an alternative build of the same library
LIB_PATH = os.environ.get("MGV_LIB_PATH") or os.path.join(_HERE, "libmugv_b200.so")
_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build the CUDA library first (make -C {_HERE}/csrc)")
        # Load torch first when it is installed: its bundled libnccl.so.2 (2.28) then satisfies our
        # libnccl.so.2 dependency, instead of the older system copy that torch cannot run against.
        try:
            import torch  # noqa: F401
        except ImportError:
            pass
        _lib = ctypes.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


def _declare(L):
    P, I, I64, F, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_float, ctypes.c_double
    L.mgv_dev_gemm.argtypes = [I, P, I64, I, P, I64, I, I, I, I, P, I64, F, I, P]
    L.mgv_dev_gemm.restype = I
    L.mgv_dev_set_gemm_mode.argtypes = [I]
    L.mgv_dev_set_fusions.argtypes = [I]
    from . import capi
    capi.declare(L)
