"""Single-core sweep of the REFERENCE CPU path (oracle/_ref: the unmodified reference sources) on the host it runs on,
per BASELINE.md's CPU-baseline plan / SURVEY 8(d):

  * 10B dims (paper_config depth 1, text 64 x 4096): forward at N in {64, 256, 512, 1024, 2048}, fwd+bwd+AdamW at
    N in {64, 256};
  * the tiny configs[0] block (H256, 4 heads, latent 4x8x8 -> 64 tokens): fwd and fwd+bwd+AdamW;
  * each job in its own process pinned to its own core (taskset -c k), so the jobs run side by side;
  * fit t = a N + b N^2 to the forward points and report the extrapolations to N = 10,920 and 57,600, LABELLED
    extrapolated (57,600 cannot run: the reference materialises 637 GB of fp64 attention probabilities).

Usage: python tools/cpu_sweep.py OUT.json
"""
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GRIDS = {64: (4, 8, 8), 256: (4, 16, 16), 512: (8, 16, 16), 1024: (16, 16, 16), 2048: (8, 32, 32)}
GRIDS_H288 = {2048: (8, 32, 32), 4096: (16, 32, 32), 8192: (16, 32, 64)}
JOBS = [("10b", "fwd", n) for n in (2048, 1024, 512, 256, 64)] + [("10b", "step", 256), ("10b", "step", 64),
                                                                    ("tiny", "fwd", 64), ("tiny", "step", 64)] + \
    [("h288", "fwd", n) for n in (8192, 4096, 2048)]


def job(args):
    core, (cfgname, kind, n) = args
    os.sched_setaffinity(0, {core})
    from oracle import oracle as O
    if cfgname == "10b":
        cfg, L = O.paper_config(depth=1), 64
        gs = O.gate_std_for(cfg.hidden)
        gate = (gs, gs / 4)
    elif cfgname == "h288":  # attention-dominated: the N^2 coefficient (head_dim 144 long-N probe)
        cfg, L = O.DitConfig(depth=1, hidden=288, heads=2, text_dim=64, c_z=24, rope_split=(48, 48, 48)), 8
        gs = O.gate_std_for(288)
        gate = (gs, gs / 4)
    else:
        cfg, L = O.DitConfig(depth=1, hidden=256, heads=4, text_dim=32, c_z=24, rope_split=(22, 22, 20)), 16
        gate = (0.2, 0.05)
    ref = O.RefModel(cfg, 1, 2, *gate)
    g = O.Rng(3).uniform_tensor((GRIDS_H288 if cfgname == "h288" else GRIDS)[n] + (cfg.c_z,), -1.0, 1.0)
    s = O.make_batch([g], 0.0, O.Rng(5))
    text = O.Rng(4).normal_tensor((L, cfg.text_dim))
    opt = O.RefAdamW(1e-4) if kind == "step" else None
    t0 = time.perf_counter()
    out = ref.flow_fwdbwd(s, text, 8.0, grads=kind == "step", with_V=False)
    if opt is not None:
        opt.update_model(ref, out["grads"])  # FlowTrainer::step (flowtrain.cpp:257-282)
    dt = time.perf_counter() - t0
    return {"config": cfgname, "kind": kind, "N": n, "seconds": dt, "core": core}


def main():
    out_path = sys.argv[1]
    from bench import host_info
    ncpu = os.cpu_count() or 1
    jobs = list(enumerate(JOBS))
    jobs = [((k + 1) % ncpu, j) for k, j in jobs]  # core 0 stays free for the bench's own cpu_baseline
    t0 = time.time()
    try:
        avail_gb = int(open("/proc/meminfo").read().split("MemAvailable:")[1].split()[0]) / 1e6
    except Exception:
        avail_gb = 64.0
    with mp.get_context("spawn").Pool(max(1, min(len(jobs), ncpu, int(avail_gb // 14)))) as pool:
        res = pool.map(job, jobs, chunksize=1)
    import numpy as np
    # the N^2 (attention) coefficient from the attention-dominated H288 points, scaled by width (4 N^2 H flops);
    # the linear coefficient from the 10B-width points with that N^2 term removed (at N <= 2048 and H = 3456 the
    # attention is < 8% of the forward, so a joint fit cannot resolve it)
    h288 = sorted((r["N"], r["seconds"]) for r in res if r["config"] == "h288")
    A = np.array([[n, n * n] for n, _ in h288], dtype=float)
    (a288, b288), *_ = np.linalg.lstsq(A, np.array([t for _, t in h288]), rcond=None)
    b = max(b288, 0.0) * 3456.0 / 288.0
    fwd = sorted((r["N"], r["seconds"]) for r in res if r["config"] == "10b" and r["kind"] == "fwd")
    a = float(np.mean([(t - b * n * n) / n for n, t in fwd]))
    steps = {r["N"]: r["seconds"] for r in res if r["config"] == "10b" and r["kind"] == "step"}
    fwds = dict(fwd)
    ratio = sum(steps[n] / fwds[n] for n in steps) / len(steps)
    ext = {}
    for n in (10920, 57600):
        tf = a * n + b * n * n
        ext[str(n)] = {"fwd_s": tf, "fwd_tokens_per_s": n / tf, "step_s": ratio * tf,
                       "step_tokens_per_s": n / (ratio * tf), "label": "EXTRAPOLATED from the fit (not run)"}
    doc = {"source": "tools/cpu_sweep.py: reference (oracle/_ref) single-threaded, one pinned core per job",
           "host": host_info(), "wall_s": time.time() - t0, "points": res,
           "fit": {"model": "t_fwd = a N + b N^2 (10B dims depth 1, text 64x4096); b from the H288 points x 3456/288",
                   "a_s_per_token": a, "b_s_per_token2": b, "b_h288": b288, "a_h288": a288, "step_over_fwd": ratio},
           "extrapolated": ext}
    with open(out_path, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc["fit"]), json.dumps(ext))


if __name__ == "__main__":
    main()
