"""profiles/kernel_traffic.json from an ncu launch list of one bench step (tools/profile_step.py):
DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch of the bench's timed phases.
  attn_fwd = the self-attention forward kernel + its V^T transpose
  attn_bwd = the self-attention backward: Q^T/K^T/V^T/dO^T transposes, D = rowsum(dO o O), dK/dV, dQ
usage: python tools/traffic_from_ncu.py launches.csv > profiles/kernel_traffic.json"""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, mi, vi, ii, gi = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Grid Size"))
per = collections.OrderedDict()
for r in rows[h + 1:]:
    if len(r) > vi:
        per.setdefault((r[ii], r[ki], r[gi]), {})[r[mi]] = float(r[vi].replace(",", ""))
big = [(k, v) for k, v in per.items() if "(54, 900, 1)" in k[2] or "attn" in k[1]]
by = lambda v: v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
# the self-attention launches are the full-grid ones (450 x 24 / 225 x 24); the backward phase is the last
# group of 4 full-size transposes + dvec + dkv + dq in the launch order
fwd = [v for k, v in big if "attn_fwd" in k[1] and "(225, 24" in k[2]]
bwd_idx = [i for i, (k, v) in enumerate(big) if "attn_bwd_dkv" in k[1] and "(450, 24" in k[2]][0]
bwd = [v for k, v in big[bwd_idx - 5:bwd_idx + 2]]
parts = {k[1].split("(")[0].split("<")[0].replace("void ", "").strip(): by(v) for k, v in big[bwd_idx - 5:bwd_idx + 2]}
fwd_t = [v for k, v in big[:big.index(next(x for x in big if "attn_fwd" in x[0][1]))] if "(54, 900" in k[2]]
out = {"attn_fwd": by(fwd[0]) + (by(fwd_t[-1]) if fwd_t else 0.0), "attn_bwd": sum(by(v) for v in bwd),
       "attn_bwd_parts": parts,
       "unit": "bytes per launch (DRAM read + write, ncu, cold cache)", "source": sys.argv[1]}
print(json.dumps(out, indent=1))
