"""profiles/kernel_traffic.json from an ncu launch list of one bench step (tools/profile_step.py):
DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch of the bench's timed phases.
  attn_fwd = the self-attention forward kernel + its V^T transpose
  attn_bwd = the self-attention backward: D = rowsum(dO o O), dK/dV, dQ (+ operand transposes, if launched)
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
big = [(k, v) for k, v in per.items() if "(54, 900, 1)" in k[2] or "attn" in k[1] or "transpose" in k[1]]
by = lambda v: v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
name = lambda k: k[1].split("(")[0].split("<")[0].replace("void ", "").replace("mgv::", "").strip()
# the self-attention launches are the full-grid ones (450 x 24 / 225 x 24).  Backward phase: D = rowsum(dO o O), dK/dV,
# dQ, plus any operand transposes launched right before it (none when the GEMM epilogues write them transposed)
fwd_i = next(i for i, (k, v) in enumerate(big) if "attn_fwd" in k[1] and "(225, 24" in k[2])
fwd = [big[fwd_i][1]] + ([big[fwd_i - 1][1]] if fwd_i and "transpose" in big[fwd_i - 1][0][1] else [])
bi = next(i for i, (k, v) in enumerate(big) if "attn_bwd_dkv" in k[1] and "(450, 24" in k[2])
lo = bi - 1
while lo > 0 and ("transpose" in big[lo - 1][0][1]):
    lo -= 1
grp = big[lo:bi + 2]
parts = {}
for k, v in grp:
    parts[name(k)] = parts.get(name(k), 0.0) + by(v)
out = {"attn_fwd": sum(by(v) for v in fwd), "attn_bwd": sum(by(v) for k, v in grp), "attn_bwd_parts": parts,
       "attn_bwd_algorithmic": None,
       "unit": "bytes per launch (DRAM read + write, ncu, cold cache)", "source": sys.argv[1]}
print(json.dumps(out, indent=1))
