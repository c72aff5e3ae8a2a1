"""Generate the committed golden fixtures from the REFERENCE ITSELF.

Run in the build container (needs /root/reference, via oracle/_ref/libmugv_ref.so):

    make -C oracle && python tests/golden/make_golden.py

Each fixture is a compressed .npz holding the case definition (config, seeds,
geometry) plus the reference's outputs for ``FlowTrainer::step`` minus AdamW
(flowtrain.cpp:257-279): the loss, per-sample velocity rows V, per-tap norms and
sampled entries, and per-parameter gradient norms and sampled entries (full
gradients for the tiny case).  Weights and inputs are NOT stored: they are
regenerated bit-exactly from the seeds by the oracle's restated Rng
(oracle/mugv_oracle.c), which test_oracle.py pins against the reference.
"""
import json
import zlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

CASES = {
    # proj/tests/test_dit.cpp tiny_config (H12, 2 heads, depth 2), two samples, one first-frame conditioned
    "tiny": dict(cfg=dict(depth=2, hidden=12, heads=2, text_dim=6, c_z=2, rope_split=(2, 2, 2)),
                 grids=[(2, 4, 4), (1, 4, 6)], L=3, mask_prob=0.5, force_cond=[0], gate_std=0.2, full=True),
    # BASELINE.json configs[0]: H256, 4 heads, 4x8x8 latent -> 64 tokens, depth 1
    "cfg0": dict(cfg=dict(depth=1, hidden=256, heads=4, text_dim=32, c_z=24, rope_split=(22, 22, 20)),
                 grids=[(4, 8, 8)], L=16, mask_prob=0.0, force_cond=[0], gate_std=0.2, full=False),
    # head_dim 144 with the paper rope split (48,48,48), 2 heads, depth 2, two samples
    "hd144": dict(cfg=dict(depth=2, hidden=288, heads=2, text_dim=64, c_z=24, rope_split=(48, 48, 48)),
                  grids=[(2, 4, 8), (3, 2, 4)], L=8, mask_prob=0.0, force_cond=[1], gate_std=O.gate_std_for(288) * 4,
                  full=False),
}
# Larger cases (SURVEY 8(c) parity plan items 2 and 4), fixtures sampled rather than full:
LONG_CASES = {
    # the benchmarked 10B width (paper_config depth 1: H3456, 24 x 144, text 64 x 4096), latent (4,8,8) -> 64 tokens,
    # first-frame conditioning on
    "w10b": dict(cfg=dict(depth=1, hidden=3456, heads=24, text_dim=4096, c_z=24, rope_split=(48, 48, 48)),
                 grids=[(4, 8, 8)], L=64, mask_prob=0.0, force_cond=[0], gate_std=O.gate_std_for(3456), full=False),
    # long N at reduced width: H288 = 2 x 144, rope (48,48,48), the 480p/2s latent (7,60,104) -> 10,920 tokens on
    # the real 480p coordinates (the reference's Tape::mha keeps 1.9 GB of probabilities; ~9 min on one core)
    "long480p": dict(cfg=dict(depth=1, hidden=288, heads=2, text_dim=64, c_z=24, rope_split=(48, 48, 48)),
                     grids=[(7, 60, 104)], L=8, mask_prob=0.0, force_cond=[0], gate_std=O.gate_std_for(288) * 4,
                     full=False),
}
ALL_CASES = dict(CASES, **LONG_CASES)
SEEDS = dict(params=1, gates=2, latents=3, text=4, batch=5)
NSAMP = 64


def build_case(name, spec):
    cfg = O.DitConfig(**spec["cfg"])
    gs = spec["gate_std"]
    P = O.open_gates(O.init_dit_params(cfg, O.Rng(SEEDS["params"])), SEEDS["gates"], gs, gs / 4)
    g = O.Rng(SEEDS["latents"])
    grids = [g.uniform_tensor((U, h, w, cfg.c_z), -1.0, 1.0) for (U, h, w) in spec["grids"]]
    text = O.Rng(SEEDS["text"]).normal_tensor((spec["L"], cfg.text_dim))
    samples = O.make_batch(grids, spec["mask_prob"], O.Rng(SEEDS["batch"]))
    for i in spec["force_cond"]:
        samples[i].cond = True
    return cfg, P, text, samples


def sample_idx(n, k, seed):
    r = np.random.default_rng(seed)
    return np.sort(r.choice(n, size=min(n, k), replace=False))


def main(names=None):
    out_dir = os.path.dirname(os.path.abspath(__file__))
    for name, spec in ALL_CASES.items():
        if names and name not in names:
            continue
        cfg, P, text, samples = build_case(name, spec)
        gs = spec["gate_std"]
        ref = O.RefModel(cfg, SEEDS["params"], SEEDS["gates"], gs, gs / 4)
        rp = ref.params()
        assert all(np.array_equal(rp[k], P[k].ravel()) for k in P), "restated Rng/init diverged from reference"
        r = ref.flow_fwdbwd(samples, text, 8.0, grads=True, with_taps=True)
        d = {"spec": np.array(json.dumps(dict(spec, seeds=SEEDS))), "loss": np.array(r["loss"])}
        for i, s in enumerate(samples):
            if spec["full"] or r["V"][i].size <= 8192:
                d[f"V.{i}"] = r["V"][i]
            else:  # sampled entries + the max |V| (normwise denominators) + the norm
                vi = sample_idx(r["V"][i].size, 4096, 200 + i)
                d[f"Vi.{i}"] = vi
                d[f"Vv.{i}"] = r["V"][i].ravel()[vi]
                d[f"Vmax.{i}"] = np.array(np.abs(r["V"][i]).max())
                d[f"Vn.{i}"] = np.array(np.linalg.norm(r["V"][i]))
            d[f"cond.{i}"] = np.array(s.cond)
            taps = r["taps"][i]
            idx = sample_idx(taps.size, 4 * NSAMP, 100 + i)
            d[f"taps_idx.{i}"] = idx
            d[f"taps_val.{i}"] = taps[idx]
            d[f"taps_norm.{i}"] = np.array(np.linalg.norm(taps))
        for k, gv in r["grads"].items():
            if spec["full"]:
                d[f"g:{k}"] = gv
            else:
                idx = sample_idx(gv.size, NSAMP, zlib.crc32(k.encode()) % 1000)
                d[f"gi:{k}"] = idx
                d[f"gv:{k}"] = gv[idx]
                d[f"gn:{k}"] = np.array(np.linalg.norm(gv))
                d[f"gm:{k}"] = np.array(np.abs(gv).max())
        path = os.path.join(out_dir, f"{name}.npz")
        np.savez_compressed(path, **d)
        print(name, "loss", r["loss"], "->", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main(sys.argv[1:] or None)
