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
          6: "NcclError", 7: "InternalError", 8: "CheckpointError", 9: "SchedulingError"}


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

class SchedulingError(MugvError):
    pass


_EXC = {1: DimensionError, 2: ConfigError, 3: InputError, 4: NumericError, 9: SchedulingError}


class mgv_dit_cfg(ctypes.Structure):
    _fields_ = [("depth", I64), ("hidden", I64), ("heads", I64), ("text_dim", I64), ("c_z", I64),
                ("rope_split", ctypes.c_int32 * 3), ("text_vocab", I64), ("text_max_len", I64)]


class mgv_flow_sample(ctypes.Structure):
    _fields_ = [("dims", I64 * 3), ("coords", P), ("clean_rows", P), ("noise", P), ("t", D), ("conditioned", P),
                ("condition_latents", P)]


class mgv_eval_sample(ctypes.Structure):
    _fields_ = [("s", mgv_flow_sample), ("text", P), ("L", I64), ("fps", D)]


class mgv_post_cfg(ctypes.Structure):
    _fields_ = [("beta", D), ("alpha_sft", D), ("gamma_merge", D), ("w_d", D), ("w_u", D), ("n_interleave", I64),
                ("interleave", P)]


class mgv_sample_record(ctypes.Structure):
    _fields_ = [("dims", I64 * 3), ("coords", P), ("rows", P), ("conditioned", P), ("condition_latents", P),
                ("text", P), ("L", I64), ("fps", D)]


class mgv_pref_pair(ctypes.Structure):
    _fields_ = [("winner", mgv_sample_record), ("loser", mgv_sample_record)]


class mgv_labeled_sample(ctypes.Structure):
    _fields_ = [("sample", mgv_sample_record), ("desirable", I)]


class mgv_post_metrics(ctypes.Structure):
    _fields_ = [("total", D), ("preference", D), ("sft", D), ("grad_norm", D)]


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
    L.mgv_rng_uniform_fill.argtypes = [ctypes.c_uint64, I64, D, D, P]
    L.mgv_make_flow_sample.argtypes = [ctypes.c_uint64, I64, I64, D, P, P, P]
    L.mgv_velocity_graph.argtypes = [P, P, I64, P, P, P, I64, P, D, P, P, P, P]
    L.mgv_plan_rank_bytes.argtypes = [ctypes.POINTER(mgv_dit_cfg), I, I, I64, I64, I64, I, P]
    L.mgv_ctx_memory.argtypes = [P, P]
    L.mgv_ctx_set_varlen.argtypes = [P, I]
    L.mgv_ctx_set_recompute.argtypes = [P, I]
    L.mgv_params_init.argtypes = [P, ctypes.POINTER(mgv_dit_cfg), ctypes.c_uint64, ctypes.c_uint64, D, D]
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
    L.mgv_prof_entry_work.argtypes = [P, I64]
    L.mgv_prof_entry_work.restype = D
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
    L.mgv_tokenize.argtypes = [ctypes.c_char_p, I64, P, I64]
    L.mgv_tokenize.restype = I64
    L.mgv_text_embed.argtypes = [P, P, I64, P, I64, P, I64, I64, P, ctypes.POINTER(I)]
    L.mgv_text_embed.restype = I
    L.mgv_patchify.argtypes = [P, P, I64, I64, I64, I64, P, P]
    L.mgv_patchify.restype = I
    L.mgv_unpatchify.argtypes = [P, P, I64, P, P, P]
    L.mgv_unpatchify.restype = I
    L.mgv_global_embed.argtypes = [P, P, I64, D, P, P]
    L.mgv_global_embed.restype = I
    L.mgv_fused_modulate.argtypes = [P, P, P, I64, P, I64, P, I64, P, I64, I64, P]
    L.mgv_fused_modulate.restype = I
    L.mgv_dev_fused_modulate_f32.argtypes = [P, P, P, P, P, P, I64, I64, P]
    L.mgv_dev_fused_modulate_f32.restype = I
    L.mgv_apply_rope3d.argtypes = [P, P, I64, I64, P, P, D, I, P]
    L.mgv_apply_rope3d.restype = I
    L.mgv_flow_errors.argtypes = [P, I64, P, P]
    L.mgv_flow_errors.restype = I
    L.mgv_flow_step_weighted.argtypes = [P, I64, P, P, P, ctypes.POINTER(D), ctypes.POINTER(D), P]
    L.mgv_flow_step_weighted.restype = I
    L.mgv_post_validate.argtypes = [P, ctypes.c_char_p, I64]
    L.mgv_post_validate.restype = I
    L.mgv_post_state_create.argtypes = [P, P, D, ctypes.c_uint64, ctypes.POINTER(P)]
    L.mgv_post_state_create.restype = I
    L.mgv_post_state_destroy.argtypes = [P]
    L.mgv_post_state_destroy.restype = None
    L.mgv_post_plan_pos.argtypes = [P]
    L.mgv_post_plan_pos.restype = I64
    L.mgv_post_last_error.argtypes = [P]
    L.mgv_post_last_error.restype = ctypes.c_char_p
    L.mgv_post_train_step.argtypes = [P, P, ctypes.c_char_p, I64, P, I64, P, I64, P, P, I64, D, P]
    L.mgv_post_train_step.restype = I
    L.mgv_post_pref_loss.argtypes = [P, P, P, ctypes.c_char_p, I64, P, I64, P, ctypes.c_uint64, ctypes.POINTER(D)]
    L.mgv_post_pref_loss.restype = I
    L.mgv_rdpo_pairs.argtypes = [P, I64, P, I64, ctypes.c_uint64, P, P]
    L.mgv_rdpo_pairs.restype = I
    L.mgv_merge_weights.argtypes = [I64, D, P]
    L.mgv_merge_weights.restype = I
    L.mgv_anneal_lr.argtypes = [I64, D, D, I64, ctypes.POINTER(D)]
    L.mgv_anneal_lr.restype = I
    L.mgv_dpo_from_errors.argtypes = [D, D, D, D, D]
    L.mgv_dpo_from_errors.restype = D
    L.mgv_kto_from_rewards.argtypes = [I64, P, P, D, D, P, ctypes.POINTER(D)]
    L.mgv_kto_from_rewards.restype = I
    L.mgv_dev_attn_fwd.restype = I
    L.mgv_dev_attn_bwd.restype = I


# symbols include/mugv_b200.h declares (checked by tests/test_capi.py)
EXPORTS = ["mgv_ctx_create", "mgv_ctx_destroy", "mgv_last_error", "mgv_ctx_set_stream", "mgv_nccl_unique_id",
           "mgv_ctx_set_dp", "mgv_ctx_set_tp", "mgv_sample_rows", "mgv_ctx_set_adamw", "mgv_adamw_steps", "mgv_param_download",
           "mgv_params_upload", "mgv_params_init", "mgv_ctx_set_varlen", "mgv_ctx_set_recompute", "mgv_plan_rank_bytes", "mgv_ctx_memory", "mgv_rng_uniform_fill", "mgv_make_flow_sample", "mgv_param_count",
           "mgv_param_name", "mgv_param_numel",
           "mgv_predict_velocity", "mgv_velocity_graph", "mgv_dit_forward", "mgv_flow_step", "mgv_flow_loss", "mgv_latent_rows",
           "mgv_rows_to_grid", "mgv_flow_step_device", "mgv_last_step_ms", "mgv_last_step_launches",
           "mgv_prof_enable", "mgv_prof_count", "mgv_prof_entry", "mgv_prof_entry_work",
           "mgv_ckpt_last_error", "mgv_ckpt_last_error_kind", "mgv_ckpt_load", "mgv_ckpt_free", "mgv_ckpt_count",
           "mgv_ckpt_name", "mgv_ckpt_dtype", "mgv_ckpt_rank", "mgv_ckpt_shape", "mgv_ckpt_numel", "mgv_ckpt_find",
           "mgv_ckpt_read", "mgv_ckpt_meta_count", "mgv_ckpt_meta_key", "mgv_ckpt_meta_value", "mgv_ckpt_save",
           "mgv_params_upload_ckpt", "mgv_params_save",
           "mgv_patchify", "mgv_unpatchify", "mgv_global_embed", "mgv_fused_modulate", "mgv_dev_fused_modulate_f32",
           "mgv_apply_rope3d", "mgv_tokenize", "mgv_text_embed",
           "mgv_flow_errors", "mgv_flow_step_weighted", "mgv_post_validate", "mgv_post_state_create",
           "mgv_post_state_destroy", "mgv_post_plan_pos", "mgv_post_last_error", "mgv_post_train_step",
           "mgv_post_pref_loss", "mgv_dpo_from_errors", "mgv_kto_from_rewards", "mgv_rdpo_pairs",
           "mgv_merge_weights", "mgv_anneal_lr"]


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


MEMORY_KEYS = ("params", "grads", "adamw", "workspace", "exchange")


def plan_rank_bytes(cfg, precision: str, tp: int, N: int, L: int, n_u: int = 2, train: bool = True,
                    recompute: bool = False) -> dict:
    """mgv_plan_rank_bytes: bytes one TP rank allocates for a step (no device needed); recompute: a training step with
    per-block activation recompute."""
    out = (I64 * 5)()
    c = cfg.to_c()
    flags = (3 if recompute else 1) if train else 0
    st = _lib().mgv_plan_rank_bytes(ctypes.byref(c), 1 if precision == "bf16" else 0, tp, N, L, n_u, flags, out)
    if st != 0:
        raise ConfigError(f"mgv_plan_rank_bytes failed ({st})")
    return dict(zip(MEMORY_KEYS, list(out)))


def rng_uniform(seed: int, shape, lo: float, hi: float) -> np.ndarray:
    """mgv_rng_uniform_fill: mugv::Rng(seed).uniform_tensor(shape, lo, hi) (the reference's stream)."""
    out = np.empty(shape, dtype=np.float64)
    st = _lib().mgv_rng_uniform_fill(seed, out.size, lo, hi, out.ctypes.data)
    if st != 0:
        raise InputError("mgv_rng_uniform_fill")
    return out


def make_flow_sample(seed: int, N: int, D: int, mask_prob: float = 0.0):
    """mgv_make_flow_sample: flow::make_batch's draws for one sample from Rng(seed) -> (noise, t, conditioned)."""
    noise = np.empty((N, D), dtype=np.float64)
    t, c = ctypes.c_double(), ctypes.c_int()
    st = _lib().mgv_make_flow_sample(seed, N, D, mask_prob, noise.ctypes.data, ctypes.byref(t), ctypes.byref(c))
    if st != 0:
        raise InputError("mgv_make_flow_sample")
    return noise, t.value, bool(c.value)


@dataclass
class FlowSample:
    """flow::FlowSample (flowtrain.hpp:111-117); rows already patchified."""
    dims: tuple
    coords: np.ndarray
    clean_rows: np.ndarray
    noise: np.ndarray
    t: float
    conditioned: np.ndarray | None = None  # (N,) uint8 unit-aligned condition mask, or None
    condition_latents: np.ndarray | None = None  # (N, D) rows for conditioned tokens; None = clean_rows
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
            if self.condition_latents is None:
                s.condition_latents = cl.ctypes.data  # first_frame_mask (flowtrain.cpp:58)
            else:
                lat = _f64(self.condition_latents)
                self._keep.append(lat)
                s.condition_latents = lat.ctypes.data
        return s


@dataclass
class SampleRecord:
    """post::SampleRecord (posttrain.hpp:15-21): latent rows on a grid, first-frame mask or none, text, fps."""
    dims: tuple
    coords: np.ndarray
    rows: np.ndarray
    text: np.ndarray
    fps: float = 8.0
    conditioned: np.ndarray | None = None
    _keep: list = field(default_factory=list, repr=False)

    def to_c(self):
        r = mgv_sample_record()
        for i in range(3):
            r.dims[i] = int(self.dims[i])
        co = np.ascontiguousarray(self.coords, dtype=np.int32)
        rw, tx = _f64(self.rows), _f64(self.text)
        self._keep = [co, rw, tx]
        r.coords, r.rows, r.text, r.L, r.fps = co.ctypes.data, rw.ctypes.data, tx.ctypes.data, tx.shape[0], self.fps
        if self.conditioned is not None and np.any(self.conditioned):
            m = np.ascontiguousarray(self.conditioned, dtype=np.uint8)
            self._keep.append(m)
            r.conditioned = m.ctypes.data
        return r


@dataclass
class PostTrainConfig:
    """post::PostTrainConfig (posttrain.hpp:37-44)."""
    beta: float = 1.0
    alpha_sft: float = 1.0
    gamma_merge: float = 0.9
    w_d: float = 1.0
    w_u: float = 1.0
    interleave: tuple = ("dpo", "kto")

    def to_c(self):
        c = mgv_post_cfg(self.beta, self.alpha_sft, self.gamma_merge, self.w_d, self.w_u, len(self.interleave), None)
        self._tags = (ctypes.c_char_p * max(1, len(self.interleave)))(*[t.encode() for t in self.interleave])
        c.interleave = ctypes.cast(self._tags, P)
        return c


def _pairs_c(pairs):
    arr = (mgv_pref_pair * max(1, len(pairs)))()
    for i, (w, l) in enumerate(pairs):
        arr[i].winner, arr[i].loser = w.to_c(), l.to_c()
    return arr


def _labels_c(labels):
    arr = (mgv_labeled_sample * max(1, len(labels)))()
    for i, (rec, desirable) in enumerate(labels):
        arr[i].sample, arr[i].desirable = rec.to_c(), int(bool(desirable))
    return arr


def tokenize(prompt: str, vocab: int) -> np.ndarray:
    """dit::tokenize (dit.cpp:193-211)."""
    L = _lib()
    n = L.mgv_tokenize(prompt.encode(), vocab, None, 0)
    ids = np.empty(max(n, 1), dtype=np.int64)
    L.mgv_tokenize(prompt.encode(), vocab, ids.ctypes.data, n)
    return ids[:n]


def merge_weights(k: int, gamma: float) -> np.ndarray:
    """post::merge_weights (posttrain.cpp:51-63)."""
    out = np.empty(max(k, 1))
    st = _lib().mgv_merge_weights(k, gamma, out.ctypes.data)
    if st != 0:
        raise _EXC.get(st, MugvError)(st, "merge_weights")
    return out[:k]


def anneal_lr(step: int, lr_start: float = 1e-4, lr_end: float = 1e-6, steps: int = 1000) -> float:
    """post::anneal_lr (posttrain.cpp:84-94)."""
    out = D()
    st = _lib().mgv_anneal_lr(step, lr_start, lr_end, steps, ctypes.byref(out))
    if st != 0:
        raise _EXC.get(st, MugvError)(st, "anneal_lr")
    return out.value


def rdpo_pairs(ctx: "Context", records, steps: int, seed: int):
    """post::rdpo_pairs on the device sampler: [(winner_rows, loser_rows)] per SampleRecord."""
    n = len(records)
    arr = (mgv_sample_record * max(1, n))(*[r.to_c() for r in records])
    outs = [(np.empty((r.rows.shape[0], ctx.cfg.patch_dim)), np.empty((r.rows.shape[0], ctx.cfg.patch_dim)))
            for r in records]
    wp = (P * max(1, n))(*[w.ctypes.data for w, _ in outs])
    lp = (P * max(1, n))(*[l.ctypes.data for _, l in outs])
    ctx._check(_lib().mgv_rdpo_pairs(ctx.h, n, arr, steps, seed, wp, lp))
    return outs


def dpo_from_errors(e_th_w, e_th_l, e_ref_w, e_ref_l, beta):
    return _lib().mgv_dpo_from_errors(e_th_w, e_th_l, e_ref_w, e_ref_l, beta)


def kto_from_rewards(rewards, desirable, w_d, w_u, z0=None):
    r = _f64(rewards)
    d = np.ascontiguousarray(desirable, dtype=np.uint8)
    z = D(z0) if z0 is not None else None
    out = D()
    st = _lib().mgv_kto_from_rewards(len(r), r.ctypes.data, d.ctypes.data, w_d, w_u,
                                     ctypes.byref(z) if z is not None else None, ctypes.byref(out))
    if st != 0:
        raise _EXC.get(st, MugvError)(st, "kto_from_rewards")
    return out.value


class PostTrainState:
    """post::PostTrainState (posttrain.hpp:128-136): `policy` is trained, `ref` holds the frozen start weights."""

    def __init__(self, policy: "Context", ref: "Context", lr: float = 1e-4, seed: int = 0):
        self._L, self.policy, self.ref = _lib(), policy, ref
        h = P()
        st = self._L.mgv_post_state_create(policy.h, ref.h, lr, seed, ctypes.byref(h))
        if st != 0:
            policy._check(st)
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self._L.mgv_post_state_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def plan_pos(self) -> int:
        return self._L.mgv_post_plan_pos(self.h)

    def train_step(self, cfg: PostTrainConfig, tag: str, pairs=(), labels=(), sft=(), sft_text=None, sft_fps=8.0):
        """post_train_step: pairs = [(winner, loser) SampleRecords], labels = [(SampleRecord, desirable)],
        sft = [FlowSample] sharing sft_text / sft_fps.  Returns dict(total, preference, sft, grad_norm)."""
        c = cfg.to_c()
        pc, lc = _pairs_c(list(pairs)), _labels_c(list(labels))
        sc = (mgv_flow_sample * max(1, len(sft)))(*[s.to_c() for s in sft])
        tx = _f64(sft_text) if sft_text is not None else None
        m = mgv_post_metrics()
        st = self._L.mgv_post_train_step(self.h, ctypes.byref(c), tag.encode(), len(pairs), pc, len(labels), lc,
                                         len(sft), sc, tx.ctypes.data if tx is not None else None,
                                         tx.shape[0] if tx is not None else 0, sft_fps, ctypes.byref(m))
        if st != 0:
            raise _EXC.get(st, MugvError)(st, self._L.mgv_post_last_error(self.h).decode())
        return {"total": m.total, "preference": m.preference, "sft": m.sft, "grad_norm": m.grad_norm}


def post_pref_loss(policy: "Context", ref: "Context", cfg: PostTrainConfig, tag: str, pairs=(), labels=(), seed=0):
    """dpo_loss / kto_loss (posttrain.cpp:171-177, 224-233) with draws from Rng(seed)."""
    c = cfg.to_c()
    pc, lc = _pairs_c(list(pairs)), _labels_c(list(labels))
    out = D()
    policy._check(_lib().mgv_post_pref_loss(policy.h, ref.h, ctypes.byref(c), tag.encode(), len(pairs), pc,
                                            len(labels), lc, seed, ctypes.byref(out)))
    return out.value


def _eval_c(recs):
    """recs: [(FlowSample, text, fps)] -> ctypes array of mgv_eval_sample (keeps buffers alive on the array)."""
    arr = (mgv_eval_sample * len(recs))()
    keep = []
    for i, (smp, text, fps) in enumerate(recs):
        tx = _f64(text)
        keep.append((smp, tx))
        arr[i].s, arr[i].text, arr[i].L, arr[i].fps = smp.to_c(), tx.ctypes.data, tx.shape[0], fps
    arr._keep = keep
    return arr


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

    def set_dp(self, rank: int, world: int, nccl_id: bytes | None):
        """mgv_ctx_set_dp; nccl_id None with world > 1: this context computes one rank's unreduced share."""
        buf = None if nccl_id is None else (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
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

    def set_varlen(self, on: bool = True):
        """mgv_ctx_set_varlen: pack multi-sample flow steps into one block-diagonal sequence."""
        self._check(self._L.mgv_ctx_set_varlen(self.h, int(on)))

    def set_recompute(self, on: bool = True):
        """mgv_ctx_set_recompute: per-block activation recompute in training steps."""
        self._check(self._L.mgv_ctx_set_recompute(self.h, int(on)))

    def memory(self) -> dict:
        """mgv_ctx_memory: this context's allocations in bytes."""
        out = (I64 * 5)()
        self._check(self._L.mgv_ctx_memory(self.h, out))
        return dict(zip(MEMORY_KEYS, list(out)))

    def init_params(self, cfg: DitConfig, seed: int = 1, gate_seed: int = 0, gate_std: float = 0.0,
                    gate_b_std: float = 0.0):
        """mgv_params_init: dit::init_dit_params(cfg, Rng(seed)) on the context (+ gate opening from
        Rng(gate_seed) when gate_seed != 0), bit-identical to the reference's weights."""
        c = cfg.to_c()
        self._check(self._L.mgv_params_init(self.h, ctypes.byref(c), seed, gate_seed, gate_std, gate_b_std))
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

    def velocity_graph(self, rows, coords, dims, text, timesteps, fps=8.0, taps=False, dV=None):
        """mgv_velocity_graph: velocity_rows_graph as one node -> dict(V[, taps][, grads]) (grads = the VJP with dV)."""
        rows, text, ts = _f64(rows), _f64(text), _f64(timesteps)
        co = np.ascontiguousarray(coords, dtype=np.int32)
        dm = (I64 * 3)(*[int(x) for x in dims])
        N, H, depth = rows.shape[0], self.cfg.hidden, self.cfg.depth
        V = np.empty((N, self.cfg.patch_dim))
        out = {"V": V}
        tp = None
        if taps:
            tl = [np.empty((N, H)) for _ in range(depth + 2)] + [np.empty((N, self.cfg.patch_dim))]
            tp = (P * len(tl))(*[a.ctypes.data for a in tl])
            out["taps"] = tl
        gp, dv = None, None
        if dV is not None:
            dv = _f64(dV)
            garr = [np.empty(k) for k in self.numels]
            gp = (P * len(garr))(*[a.ctypes.data for a in garr])
            out["grads"] = dict(zip(self.names, garr))
        self._check(self._L.mgv_velocity_graph(self.h, rows.ctypes.data, N, co.ctypes.data, dm, text.ctypes.data,
                                                text.shape[0], ts.ctypes.data, fps, V.ctypes.data, tp,
                                                None if dv is None else dv.ctypes.data, gp))
        return out

    def fused_modulate(self, x, bias, scale, shift, residual):
        """SPEC fused_modulate: residual + ((x + bias) * (1 + scale) + shift) on a 2-D fp64
        array; bias / scale / shift are scalars, per-channel vectors or full arrays."""
        x, res = _f64(x), _f64(residual)
        rows, cols = x.shape
        b, sc, sh = (_f64(np.asarray(a)).ravel() for a in (bias, scale, shift))
        out = np.empty_like(x)
        self._check(self._L.mgv_fused_modulate(self.h, x.ctypes.data, b.ctypes.data, b.size, sc.ctypes.data, sc.size,
                                               sh.ctypes.data, sh.size, res.ctypes.data, rows, cols, out.ctypes.data))
        return out

    def dev_fused_modulate_f32(self, x, bias, scale, shift, residual, out):
        """The fp32 device form on device pointers (torch tensors or raw addresses), asynchronous on the context
        stream."""
        ptr = lambda a: a if isinstance(a, int) else a.data_ptr()
        rows, cols = x.shape
        self._check(self._L.mgv_dev_fused_modulate_f32(self.h, ptr(x), ptr(bias), ptr(scale), ptr(shift),
                                                       ptr(residual), rows, cols, ptr(out)))

    def apply_rope3d(self, x, coords, split, heads, base=10000.0, inverse=False):
        """SPEC apply_rope3d = Tape::rope3d (autodiff.cpp:849-898) on x (N, heads * sum(split)) fp64."""
        x = _f64(x)
        co = np.ascontiguousarray(coords, dtype=np.int32)
        sp = (I64 * 3)(*[int(v) for v in split])
        out = np.empty_like(x)
        self._check(self._L.mgv_apply_rope3d(self.h, x.ctypes.data, x.shape[0], heads, sp, co.ctypes.data, base,
                                             1 if inverse else 0, out.ctypes.data))
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

    def latent_rows(self, grid):
        """mgv_latent_rows (dit::latent_rows): (U, h, w, C) grid -> (N, 4C) rows and (N, 3) coords."""
        g = _f64(grid)
        U, h, w, C = g.shape
        N = U * (h // 2) * (w // 2)
        rows = np.empty((N, 4 * C))
        coords = np.empty((N, 3), dtype=np.int32)
        self._check(self._L.mgv_latent_rows(self.h, g.ctypes.data, U, h, w, C, rows.ctypes.data, coords.ctypes.data))
        return rows, coords

    def rows_to_grid(self, rows, coords, dims, C):
        """mgv_rows_to_grid (dit::rows_to_grid): rows on coords of a (U, H', W') token grid -> (U, 2H', 2W', C)."""
        r = _f64(rows)
        co = np.ascontiguousarray(coords, dtype=np.int32)
        dm = (I64 * 3)(*[int(x) for x in dims])
        out = np.empty((int(dims[0]), 2 * int(dims[1]), 2 * int(dims[2]), int(C)))
        self._check(self._L.mgv_rows_to_grid(self.h, r.ctypes.data, co.ctypes.data, r.shape[0], dm, int(C),
                                             out.ctypes.data))
        return out

    def text_embed(self, ids, embed_table, null_row, max_len=64):
        """dit::text_embed: (rows (L, text_dim), truncated)."""
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        tab = _f64(embed_table)
        nul = _f64(null_row).ravel()
        L = max(1, min(len(ids), max_len))
        out = np.empty((L, tab.shape[1]))
        tr = I()
        self._check(self._L.mgv_text_embed(self.h, ids.ctypes.data if len(ids) else None, len(ids), tab.ctypes.data,
                                           tab.shape[0], nul.ctypes.data, tab.shape[1], max_len, out.ctypes.data,
                                           ctypes.byref(tr)))
        return out, bool(tr.value)

    def patchify(self, grid):
        """dit::patchify: (U, h, w, C) grid -> (tokens (N, hidden), coords (N, 3))."""
        g = _f64(grid)
        U, h, w, C = g.shape
        N = U * (h // 2) * (w // 2)
        tok = np.empty((N, self.cfg.hidden))
        coords = np.empty((N, 3), dtype=np.int32)
        self._check(self._L.mgv_patchify(self.h, g.ctypes.data, U, h, w, C, tok.ctypes.data, coords.ctypes.data))
        return tok, coords

    def unpatchify(self, tokens, coords, dims):
        """dit::unpatchify: tokens (N, hidden) on coords of dims (U, H', W') -> (U, 2H', 2W', c_z)."""
        t = _f64(tokens)
        co = np.ascontiguousarray(coords, dtype=np.int32)
        dm = (I64 * 3)(*[int(x) for x in dims])
        out = np.empty((int(dims[0]), 2 * int(dims[1]), 2 * int(dims[2]), self.cfg.c_z))
        self._check(self._L.mgv_unpatchify(self.h, t.ctypes.data, t.shape[0], co.ctypes.data, dm, out.ctypes.data))
        return out

    def global_embed(self, timesteps, fps=8.0):
        """dit::global_embed: (g (N, hidden), block_scales (depth, hidden))."""
        ts = _f64(timesteps)
        g = np.empty((ts.shape[0], self.cfg.hidden))
        bs = np.empty((self.cfg.depth, self.cfg.hidden))
        self._check(self._L.mgv_global_embed(self.h, ts.ctypes.data, ts.shape[0], fps, g.ctypes.data, bs.ctypes.data))
        return g, bs

    def flow_errors(self, recs):
        """mgv_flow_errors: post::flow_error of each (FlowSample, text, fps), forward only."""
        arr = _eval_c(recs)
        errs = np.empty(len(recs))
        self._check(self._L.mgv_flow_errors(self.h, len(recs), arr, errs.ctypes.data))
        return errs

    def flow_step_weighted(self, recs, weights, grads=False):
        """mgv_flow_step_weighted: one fwd+bwd of sum_k w_k l_k; returns dict(loss, errs, grad_norm[, grads])."""
        arr = _eval_c(recs)
        w = _f64(weights)
        errs = np.empty(len(recs))
        loss, gn = D(), D()
        g_arrs = [np.empty(k) for k in self.numels] if grads else None
        gp = (P * len(g_arrs))(*[a.ctypes.data for a in g_arrs]) if grads else None
        self._check(self._L.mgv_flow_step_weighted(self.h, len(recs), arr, w.ctypes.data, errs.ctypes.data,
                                                   ctypes.byref(loss), ctypes.byref(gn), gp))
        out = {"loss": loss.value, "errs": errs, "grad_norm": gn.value}
        if grads:
            out["grads"] = dict(zip(self.names, g_arrs))
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
            out[name] = {"ms": ms.value, "launches": n.value, "flops": self._L.mgv_prof_entry_work(self.h, i)}
        return out
