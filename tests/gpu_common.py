"""Helpers shared by the GPU parity tests: convert oracle cases to C-ABI inputs."""
import numpy as np

from oracle import oracle as O
from paper_2510_17519_b200.capi import DitConfig, FlowSample


def to_cfg(c: O.DitConfig) -> DitConfig:
    return DitConfig(depth=c.depth, hidden=c.hidden, heads=c.heads, text_dim=c.text_dim, c_z=c.c_z,
                     rope_split=tuple(c.rope_split))


def to_samples(samples):
    out = []
    for s in samples:
        m = O.condition_flags(s)
        cond = None if m is None else m.astype(np.uint8)
        out.append(FlowSample(s.dims, s.coords, s.clean, s.noise, s.t, cond,
                              None if cond is None else s.cond_latents))
    return out


def nerr(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    den = np.abs(b).max()
    if den == 0:
        return float(np.abs(a).max())
    return float(np.abs(a - b).max() / den)
