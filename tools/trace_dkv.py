"""Timeline of one dK/dV (v8) CTA from a -DMGV_ATTN_TRACE build (variants/trace): per-step event clocks.
Usage: python tools/trace_dkv.py [N]"""
import ctypes
import os
import sys

os.environ["MGV_LIB_PATH"] = "variants/trace/libmugv_b200.so"
N = sys.argv[1] if len(sys.argv) > 1 else "14400"
sys.argv = ["probe", N, "bwd", "1"]
exec(open("tools/probe_attn.py").read())
from paper_2510_17519_b200._lib import lib  # noqa: E402
buf = (ctypes.c_ulonglong * (8 * 64))()
lib().mgv_dev_attn_trace2(buf)
ev = [[buf[e * 64 + j] for j in range(64)] for e in range(8)]
t0 = ev[3][0]
t0 = ev[0][0]
names = ["mma:top", "S(i+1) iss", "p_full ok", "dV(i) iss", "ds_full ok", "dK(i) iss", "dP(i+1) iss", "cmp:S(i) ok"]
print("step " + " ".join(f"{n:>12s}" for n in names) + "   period")
for j in range(1, 24):
    row = [ev[e][j] - t0 for e in range(8)]
    print(f"{j:4d} " + " ".join(f"{v:12d}" for v in row) + f"   {ev[0][j] - ev[0][j - 1]:6d}")

# the dQ pass of the same run (events of tools/trace_attn.py)
lib().mgv_dev_attn_trace(buf)
ev = [[buf[e * 64 + j] for j in range(64)] for e in range(8)]
t0 = ev[3][0]
names = ["mma:S(j+2)", "mma:dpE(j)", "mma:dsF(j)", "cmp:S(j+1) ok", "cmp:dP ok", "cmp:math done", "cmp:dsF arrive"]
print("dQ pass")
print("step " + " ".join(f"{n:>14s}" for n in names) + "   period")
for j in range(2, 24):
    row = [ev[e][j] - t0 for e in range(7)]
    print(f"{j:4d} " + " ".join(f"{v:14d}" for v in row) + f"   {ev[3][j] - ev[3][j - 1]:6d}")
