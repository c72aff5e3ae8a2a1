"""ctypes binding of the C ABI (include/mugv_b200.h) and a thin Python mirror of
the reference's value API (proj/include/mugv/dit.hpp, flowtrain.hpp).

All compute happens in ``libmugv_b200.so`` on the GPU.  If the library is
missing, or no CUDA device is present, calls raise; there is no fallback.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from ._lib import lib as _lib

P, I, I64, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double

STATUS = {0: "OK", 1: "DimensionError", 2: "ConfigError", 3: "InputError", 4: "NumericError", 5: "CudaError",
          6: "NcclError", 7: "InternalError", 8: "CheckpointError"}


class MugvError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.kind = STATUS.get(status, str(status))


class DimensionError(MugvError):
    pass


class ConfigError(MugvError):
    pass


class InputError(MugvError):
    pass


class NumericError(MugvError):
    pass


class CheckpointError(MugvError):
    """mugv::CheckpointError (errors.hpp:41-45); .ckpt_kind is one of CKPT_KINDS."""
    def __init__(self, status, msg, kind):
        super().__init__(status, msg)
        self.ckpt_kind = kind


CKPT_KINDS = {0: "BadMagic", 1: "Truncated", 2: "BadHeader", 3: "BadOffsets", 4: "Io"}  # CheckpointError::Kind

_EXC = {1: DimensionError, 2: ConfigError, 3: InputError, 4: NumericError}


class mgv_dit_cfg(ctypes.Structure):
    _fields_ = [("depth", I64), ("hidden", I64), ("heads", I64), ("text_dim", I64), ("c_z", I64),
                ("rope_split", ctypes.c_int32 * 3), ("text_vocab", I64), ("text_max_len", I64)]


class mgv_flow_sample(ctypes.Structure):
    _fields_ = [("dims", I64 * 3), ("coords", P), ("clean_rows", P), ("noise", P), ("t", D), ("conditioned", P),
                ("condition_latents", P)]


def declare(L):
    L.mgv_ctx_create.argtypes = [I, I, ctypes.POINTER(P)]
    L.mgv_ctx_create.restype = I
    L.mgv_ctx_destroy.argtypes = [P]
    L.mgv_last_error.argtypes = [P]
    L.mgv_last_error.restype = ctypes.c_char_p
    L.mgv_ctx_set_stream.argtypes = [P, P]
    L.mgv_ctx_set_stream.restype = I
    L.mgv_nccl_unique_id.argtypes = [P]
    L.mgv_nccl_unique_id.restype = I
    L.mgv_ctx_set_dp.argtypes = [P, I, I, P]
    L.mgv_ctx_set_dp.restype = I
    L.mgv_ctx_set_tp.argtypes = [P, I, I, P]
    L.mgv_ctx_set_tp.restype = I
    L.mgv_sample_rows.argtypes = [P, P, I64, P, P, P, I64, P, P, I64, I, D, P]
    L.mgv_sample_rows.restype = I
    L.mgv_ctx_set_adamw.argtypes = [P, D, D, D, D, D]
    L.mgv_ctx_set_adamw.restype = I
    L.mgv_adamw_steps.argtypes = [P]
    L.mgv_adamw_steps.restype = I64
    L.mgv_param_download.argtypes = [P, I64, P]
    L.mgv_param_download.restype = I
    L.mgv_params_upload.argtypes = [P, ctypes.POINTER(mgv_dit_cfg), I64, P, P, P]
    L.mgv_params_upload.restype = I
    L.mgv_param_count.argtypes = [P]
    L.mgv_param_count.restype = I64
    L.mgv_param_name.argtypes = [P, I64]
    L.mgv_param_name.restype = ctypes.c_char_p
    L.mgv_param_numel.argtypes = [P, I64]
    L.mgv_param_numel.restype = I64
    L.mgv_predict_velocity.argtypes = [P, P, I64, P, P, P, I64, P, D, P]
    L.mgv_predict_velocity.restype = I
    L.mgv_dit_forward.argtypes = [P, P, I64, P, P, P, I64, P, D, P]
    L.mgv_dit_forward.restype = I
    L.mgv_flow_step.argtypes = [P, I64, ctypes.POINTER(mgv_flow_sample), P, I64, D, ctypes.POINTER(D),
                                ctypes.POINTER(D), P, P]
    L.mgv_flow_step.restype = I
    L.mgv_flow_step_device.argtypes = [P, I64, ctypes.POINTER(mgv_flow_sample), P, I64, D, ctypes.POINTER(D),
                                       ctypes.POINTER(D)]
    L.mgv_flow_step_device.restype = I
    L.mgv_flow_loss.argtypes = [P, P, P, P, I64, I64, ctypes.POINTER(D)]
    L.mgv_flow_loss.restype = I
    L.mgv_latent_rows.argtypes = [P, P, I64, I64, I64, I64, P, P]
    L.mgv_latent_rows.restype = I
    L.mgv_rows_to_grid.argtypes = [P, P, P, I64, P, I64, P]
    L.mgv_rows_to_grid.restype = I
    L.mgv_last_step_ms.argtypes = [P]
    L.mgv_last_step_ms.restype = D
    L.mgv_last_step_launches.argtypes = [P]
    L.mgv_last_step_launches.restype = I64
    L.mgv_prof_enable.argtypes = [P, I]
    L.mgv_prof_enable.restype = I
    L.mgv_prof_count.argtypes = [P]
    L.mgv_prof_count.restype = I64
    L.mgv_prof_entry.argtypes = [P, I64, ctypes.POINTER(D), ctypes.POINTER(I64)]
    L.mgv_prof_entry.restype = ctypes.c_char_p
    CP = ctypes.c_char_p
    L.mgv_ckpt_last_error.argtypes = []
    L.mgv_ckpt_last_error.restype = CP
    L.mgv_ckpt_last_error_kind.argtypes = []
    L.mgv_ckpt_last_error_kind.restype = I
    L.mgv_ckpt_load.argtypes = [CP, ctypes.POINTER(P)]
    L.mgv_ckpt_load.restype = I
    L.mgv_ckpt_free.argtypes = [P]
    L.mgv_ckpt_free.restype = None
    L.mgv_ckpt_count.argtypes = [P]
    L.mgv_ckpt_count.restype = I64
    L.mgv_ckpt_name.argtypes = [P, I64]
    L.mgv_ckpt_name.restype = CP
    L.mgv_ckpt_dtype.argtypes = [P, I64]
    L.mgv_ckpt_dtype.restype = I
    L.mgv_ckpt_rank.argtypes = [P, I64]
    L.mgv_ckpt_rank.restype = I
    L.mgv_ckpt_shape.argtypes = [P, I64]
    L.mgv_ckpt_shape.restype = ctypes.POINTER(I64)
    L.mgv_ckpt_numel.argtypes = [P, I64]
    L.mgv_ckpt_numel.restype = I64
    L.mgv_ckpt_find.argtypes = [P, CP]
    L.mgv_ckpt_find.restype = I64
    L.mgv_ckpt_read.argtypes = [P, I64, P]
    L.mgv_ckpt_read.restype = I
    L.mgv_ckpt_meta_count.argtypes = [P]
    L.mgv_ckpt_meta_count.restype = I64
    L.mgv_ckpt_meta_key.argtypes = [P, I64]
    L.mgv_ckpt_meta_key.restype = CP
    L.mgv_ckpt_meta_value.argtypes = [P, I64]
    L.mgv_ckpt_meta_value.restype = CP
    L.mgv_ckpt_save.argtypes = [CP, I64, P, P, P, P, P, I64, P, P]
    L.mgv_ckpt_save.restype = I
    L.mgv_params_upload_ckpt.argtypes = [P, ctypes.POINTER(mgv_dit_cfg), P]
    L.mgv_params_upload_ckpt.restype = I
    L.mgv_params_save.argtypes = [P, CP, I, I64, P, P]
    L.mgv_params_save.restype = I
    L.mgv_dev_attn_fwd.restype = I
    L.mgv_dev_attn_bwd.restype = I


# symbols include/mugv_b200.h declares (checked by tests/test_capi.py)
EXPORTS = ["mgv_ctx_create", "mgv_ctx_destroy", "mgv_last_error", "mgv_ctx_set_stream", "mgv_nccl_unique_id",
           "mgv_ctx_set_dp", "mgv_ctx_set_tp", "mgv_sample_rows", "mgv_ctx_set_adamw", "mgv_adamw_steps", "mgv_param_download",
           "mgv_params_upload", "mgv_param_count", "mgv_param_name", "mgv_param_numel",
           "mgv_predict_velocity", "mgv_dit_forward", "mgv_flow_step", "mgv_flow_loss", "mgv_latent_rows",
           "mgv_rows_to_grid", "mgv_flow_step_device", "mgv_last_step_ms", "mgv_last_step_launches",
           "mgv_prof_enable", "mgv_prof_count", "mgv_prof_entry",
           "mgv_ckpt_last_error", "mgv_ckpt_last_error_kind", "mgv_ckpt_load", "mgv_ckpt_free", "mgv_ckpt_count",
           "mgv_ckpt_name", "mgv_ckpt_dtype", "mgv_ckpt_rank", "mgv_ckpt_shape", "mgv_ckpt_numel", "mgv_ckpt_find",
           "mgv_ckpt_read", "mgv_ckpt_meta_count", "mgv_ckpt_meta_key", "mgv_ckpt_meta_value", "mgv_ckpt_save",
           "mgv_params_upload_ckpt", "mgv_params_save"]


# ---------------------------------------------------------------- MUGVCKPT (params.hpp:54-61)
F32, F64 = 0, 1  # Dtype (params.hpp:14)


def _ckpt_raise(st):
    L = _lib()
    msg = L.mgv_ckpt_last_error().decode(errors="replace")
    if st == 8:
        raise CheckpointError(st, msg, CKPT_KINDS.get(L.mgv_ckpt_last_error_kind(), "?"))
    raise _EXC.get(st, MugvError)(st, msg)


class Checkpoint:
    """A loaded MUGVCKPT file (mugv::load_checkpoint, params.cpp:128-225): sorted entries, host-side."""

    def __init__(self, path: str):
        L = _lib()
        h = P()
        st = L.mgv_ckpt_load(str(path).encode(), ctypes.byref(h))
        if st != 0:
            _ckpt_raise(st)
        self._L, self.h = L, h

    def close(self):
        if getattr(self, "h", None):
            self._L.mgv_ckpt_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def names(self) -> list:
        return [self._L.mgv_ckpt_name(self.h, i).decode() for i in range(self._L.mgv_ckpt_count(self.h))]

    def dtype(self, name: str) -> int:
        return self._L.mgv_ckpt_dtype(self.h, self._index(name))

    def _index(self, name: str) -> int:
        i = self._L.mgv_ckpt_find(self.h, name.encode())
        if i < 0:
            raise InputError(3, f'no parameter named "{name}"')
        return i

    def __getitem__(self, name: str) -> np.ndarray:
        i = self._index(name)
        r = self._L.mgv_ckpt_rank(self.h, i)
        sp = self._L.mgv_ckpt_shape(self.h, i)
        shape = tuple(int(sp[k]) for k in range(r))
        out = np.empty(int(self._L.mgv_ckpt_numel(self.h, i)), dtype=np.float64)
        st = self._L.mgv_ckpt_read(self.h, i, out.ctypes.data)
        if st != 0:
            _ckpt_raise(st)
        return out.reshape(shape)

    def metadata(self) -> dict:
        n = self._L.mgv_ckpt_meta_count(self.h)
        return {self._L.mgv_ckpt_meta_key(self.h, i).decode(): self._L.mgv_ckpt_meta_value(self.h, i).decode()
                for i in range(n)}

    def to_dict(self) -> dict:
        return {k: self[k] for k in self.names()}


def _meta_arrays(meta):
    keys = list(meta or {})
    ck = (ctypes.c_char_p * max(1, len(keys)))(*[k.encode() for k in keys])
    cv = (ctypes.c_char_p * max(1, len(keys)))(*[str(meta[k]).encode() for k in keys])
    return len(keys), ck, cv


def load_checkpoint(path: str) -> Checkpoint:
    return Checkpoint(path)


def save_checkpoint(path: str, params: dict, dtypes: dict | None = None, metadata: dict | None = None):
    """mugv::save_checkpoint (params.cpp:92-126): name -> array, optional name -> F32/F64, string metadata."""
    names = list(params)
    arrs = [np.ascontiguousarray(params[k], dtype=np.float64) for k in names]
    n = len(names)
    cn = (ctypes.c_char_p * max(1, n))(*[k.encode() for k in names])
    dp = (P * max(1, n))(*[a.ctypes.data for a in arrs])
    dt = (I * max(1, n))(*[int((dtypes or {}).get(k, F64)) for k in names])
    rk = (I * max(1, n))(*[a.ndim for a in arrs])
    shp = [(I64 * max(1, a.ndim))(*a.shape) for a in arrs]
    sp = (P * max(1, n))(*[ctypes.addressof(x) for x in shp])
    nm, mk, mv = _meta_arrays(metadata)
    st = _lib().mgv_ckpt_save(str(path).encode(), n, cn, dp, dt, rk, sp, nm, mk, mv)
    if st != 0:
        _ckpt_raise(st)


@dataclass
class DitConfig:
    """dit::DitConfig (proj/include/mugv/dit.hpp:13-26)."""
    depth: int = 4
    hidden: int = 64
    heads: int = 4
    text_dim: int = 32
    c_z: int = 24
    rope_split: tuple = (4, 6, 6)
    text_vocab: int = 4096
    text_max_len: int = 64

    @property
    def head_dim(self):
        return self.hidden // self.heads

    @property
    def patch_dim(self):
        return 4 * self.c_z

    def to_c(self):
        c = mgv_dit_cfg(self.depth, self.hidden, self.heads, self.text_dim, self.c_z)
        for i in range(3):
            c.rope_split[i] = self.rope_split[i]
        c.text_vocab = self.text_vocab
        c.text_max_len = self.text_max_len
        return c


def paper_config(depth=56):
    """dit.cpp:40-48: the 10B shape."""
    return DitConfig(depth=depth, hidden=3456, heads=24, text_dim=4096, c_z=24, rope_split=(48, 48, 48))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class FlowSample:
    """flow::FlowSample (flowtrain.hpp:111-117); rows already patchified."""
    dims: tuple
    coords: np.ndarray
    clean_rows: np.ndarray
    noise: np.ndarray
    t: float
    conditioned: np.ndarray | None = None  # (N,) uint8 first-frame mask, or None
    _keep: list = field(default_factory=list, repr=False)

    def to_c(self):
        s = mgv_flow_sample()
        for i in range(3):
            s.dims[i] = int(self.dims[i])
        co = np.ascontiguousarray(self.coords, dtype=np.int32)
        cl = _f64(self.clean_rows)
        nz = _f64(self.noise)
        self._keep = [co, cl, nz]
        s.coords, s.clean_rows, s.noise, s.t = co.ctypes.data, cl.ctypes.data, nz.ctypes.data, float(self.t)
        if self.conditioned is not None and np.any(self.conditioned):
            m = np.ascontiguousarray(self.conditioned, dtype=np.uint8)
            self._keep.append(m)
            s.conditioned = m.ctypes.data
            s.condition_latents = cl.ctypes.data
        return s


class Context:
    """One device, one precision ("fp32" parity mode or "bf16" tensor-core mode)."""

    def __init__(self, device: int = 0, precision: str = "bf16"):
        self._L = _lib()
        h = P()
        prec = {"fp32": 0, "bf16": 1}[precision]
        st = self._L.mgv_ctx_create(device, prec, ctypes.byref(h))
        if st != 0:
            raise MugvError(st, "mgv_ctx_create failed (no CUDA device?)")
        self.h = h
        self.precision = precision
        self.cfg = None
        self.names = []

    def close(self):
        if getattr(self, "h", None):
            self._L.mgv_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st != 0:
            msg = self._L.mgv_last_error(self.h).decode()
            if st == 8:
                raise CheckpointError(st, msg, CKPT_KINDS.get(self._L.mgv_ckpt_last_error_kind(), "?"))
            raise _EXC.get(st, MugvError)(st, msg)

    def set_stream(self, stream_ptr: int):
        self._check(self._L.mgv_ctx_set_stream(self.h, stream_ptr))

    def set_dp(self, rank: int, world: int, nccl_id: bytes):
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
        self._check(self._L.mgv_ctx_set_dp(self.h, rank, world, buf))

    def sample_rows(self, x_start, coords, dims, text, steps, direction=-1, fps=8.0, cond=None, cond_latents=None):
        """flow::forward_sample_rows (direction -1) / reverse_sample_rows (+1) on device."""
        x = _f64(x_start)
        out = np.empty_like(x)
        co = np.ascontiguousarray(coords, dtype=np.int32)
        d = np.asarray(dims, dtype=np.int64)
        tx = _f64(text)
        cm = None if cond is None else np.ascontiguousarray(cond, dtype=np.uint8)
        cl = None if cond_latents is None else _f64(cond_latents)
        self._check(self._L.mgv_sample_rows(self.h, x.ctypes.data, x.shape[0], co.ctypes.data, d.ctypes.data,
                                            tx.ctypes.data, tx.shape[0], None if cm is None else cm.ctypes.data,
                                            None if cl is None else cl.ctypes.data, steps, direction, fps,
                                            out.ctypes.data))
        return out

    def set_adamw(self, lr: float = 1e-3, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                  weight_decay: float = 0.0):
        """Run AdamW::update (optim.cpp:7-24) on device after every flow step; lr <= 0 disables."""
        self._check(self._L.mgv_ctx_set_adamw(self.h, lr, beta1, beta2, eps, weight_decay))

    def adamw_steps(self) -> int:
        return int(self._L.mgv_adamw_steps(self.h))

    def download(self) -> dict:
        """All dit.* parameters (reference layout) as fp64 arrays keyed by name."""
        out = {}
        for i in range(int(self._L.mgv_param_count(self.h))):
            name = self._L.mgv_param_name(self.h, i).decode()
            buf = np.empty(int(self._L.mgv_param_numel(self.h, i)), dtype=np.float64)
            self._check(self._L.mgv_param_download(self.h, i, buf.ctypes.data))
            out[name] = buf
        return out

    def set_tp(self, size: int, rank: int = 0, nccl_id: bytes | None = None):
        """Megatron tensor parallelism (call before upload).  nccl_id None: emulate all ranks here."""
        buf = None if nccl_id is None else (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
        self._check(self._L.mgv_ctx_set_tp(self.h, size, rank, buf))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        st = _lib().mgv_nccl_unique_id(buf)
        if st != 0:
            raise MugvError(st, "ncclGetUniqueId failed")
        return bytes(buf)

    def upload(self, cfg: DitConfig, params: dict):
        """mgv_params_upload of a dit.* ParameterSet (name -> ndarray)."""
        names = list(params)
        arrs = [_f64(params[k]).ravel() for k in names]
        cn = (ctypes.c_char_p * len(names))(*[k.encode() for k in names])
        dp = (P * len(names))(*[a.ctypes.data for a in arrs])
        ne = (I64 * len(names))(*[a.size for a in arrs])
        c = cfg.to_c()
        self._check(self._L.mgv_params_upload(self.h, ctypes.byref(c), len(names), cn, dp, ne))
        self.cfg = cfg
        self.names = [self._L.mgv_param_name(self.h, i).decode() for i in range(self._L.mgv_param_count(self.h))]
        self.numels = [self._L.mgv_param_numel(self.h, i) for i in range(len(self.names))]

    def upload_checkpoint(self, cfg: DitConfig, ck: "Checkpoint"):
        """mgv_params_upload_ckpt: the checkpoint's dit.* entries straight to the device."""
        c = cfg.to_c()
        self._check(self._L.mgv_params_upload_ckpt(self.h, ctypes.byref(c), ck.h))
        self.cfg = cfg
        self.names = [self._L.mgv_param_name(self.h, i).decode() for i in range(self._L.mgv_param_count(self.h))]
        self.numels = [self._L.mgv_param_numel(self.h, i) for i in range(len(self.names))]

    def save_checkpoint(self, path: str, dtype: int = F32, metadata: dict | None = None):
        """mgv_params_save: save_checkpoint of the device dit.* parameters."""
        nm, mk, mv = _meta_arrays(metadata)
        self._check(self._L.mgv_params_save(self.h, str(path).encode(), int(dtype), nm, mk, mv))

    def predict_velocity(self, rows, coords, dims, text, timesteps, fps=8.0):
        rows, text, ts = _f64(rows), _f64(text), _f64(timesteps)
        co = np.ascontiguousarray(coords, dtype=np.int32)
        dm = (I64 * 3)(*[int(x) for x in dims])
        out = np.empty((rows.shape[0], self.cfg.patch_dim))
        self._check(self._L.mgv_predict_velocity(self.h, rows.ctypes.data, rows.shape[0], co.ctypes.data, dm,
                                                  text.ctypes.data, text.shape[0], ts.ctypes.data, fps,
                                                  out.ctypes.data))
        return out

    def dit_forward(self, tokens, coords, dims, text, timesteps, fps=8.0):
        tokens, text, ts = _f64(tokens), _f64(text), _f64(timesteps)
        co = np.ascontiguousarray(coords, dtype=np.int32)
        dm = (I64 * 3)(*[int(x) for x in dims])
        out = np.empty((tokens.shape[0], self.cfg.hidden))
        self._check(self._L.mgv_dit_forward(self.h, tokens.ctypes.data, tokens.shape[0], co.ctypes.data, dm,
                                             text.ctypes.data, text.shape[0], ts.ctypes.data, fps, out.ctypes.data))
        return out

    def flow_step(self, samples, text, fps=8.0, grads=False, velocity=False):
        """FlowTrainer::step: forward+backward (+ AdamW::update when set_adamw is on); returns dict(loss,
        grad_norm[, grads][, V]) -- the gradients are the ones the optimizer consumed."""
        n = len(samples)
        cs = (mgv_flow_sample * n)(*[s.to_c() for s in samples])
        text = _f64(text)
        loss, gn = D(), D()
        g_arrs = None
        gp = None
        if grads:
            g_arrs = [np.empty(k) for k in self.numels]
            gp = (P * len(g_arrs))(*[a.ctypes.data for a in g_arrs])
        v_arrs = None
        vp = None
        if velocity:
            v_arrs = [np.empty((s.clean_rows.shape[0], self.cfg.patch_dim)) for s in samples]
            vp = (P * n)(*[a.ctypes.data for a in v_arrs])
        self._check(self._L.mgv_flow_step(self.h, n, cs, text.ctypes.data, text.shape[0], fps, ctypes.byref(loss),
                                           ctypes.byref(gn), gp, vp))
        out = {"loss": loss.value, "grad_norm": gn.value, "ms": self._L.mgv_last_step_ms(self.h)}
        if grads:
            out["grads"] = dict(zip(self.names, g_arrs))
        if velocity:
            out["V"] = v_arrs
        return out

    def flow_step_device(self, samples_c, text_dev_ptr, L, fps=8.0):
        """mgv_flow_step_device: samples_c is a ctypes array of mgv_flow_sample holding DEVICE pointers."""
        loss, gn = D(), D()
        self._check(self._L.mgv_flow_step_device(self.h, len(samples_c), samples_c, text_dev_ptr, L, fps,
                                                  ctypes.byref(loss), ctypes.byref(gn)))
        return loss.value, gn.value

    def last_step_ms(self) -> float:
        return self._L.mgv_last_step_ms(self.h)

    def last_step_launches(self) -> int:
        return self._L.mgv_last_step_launches(self.h)

    def prof_enable(self, on=True):
        self._check(self._L.mgv_prof_enable(self.h, 1 if on else 0))

    def prof_stats(self) -> dict:
        out = {}
        for i in range(self._L.mgv_prof_count(self.h)):
            ms, n = D(), I64()
            name = self._L.mgv_prof_entry(self.h, i, ctypes.byref(ms), ctypes.byref(n)).decode()
            out[name] = {"ms": ms.value, "launches": n.value}
        return out
