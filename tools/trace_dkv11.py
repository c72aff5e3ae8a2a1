"""Timeline of one dK/dV v11 CTA (blockIdx (7, 0)) from a -DMGV_ATTN_TRACE build: per-step event clocks.
Usage: python tools/trace_dkv11.py [N]  (MGV_LIB_PATH -> the trace build)"""
import ctypes
import os
import sys

os.environ.setdefault("MGV_LIB_PATH", "tools/trace_lib/libmugv_b200.so")
N = sys.argv[1] if len(sys.argv) > 1 else "57600"
sys.argv = ["probe", N, "bwd", "1"]
exec(open("tools/probe_attn.py").read())
from paper_2510_17519_b200._lib import lib  # noqa: E402
buf = (ctypes.c_ulonglong * (8 * 64))()
lib().mgv_dev_attn_trace2(buf)
ev = [[buf[e * 64 + j] for j in range(64)] for e in range(8)]
t0 = ev[4][0]
names = ["mma:s_loaded", "mma:p_full", "mma:dp_loaded", "mma:ds_full", "cmp:s_full", "cmp:p_full>", "cmp:dp_full",
         "cmp:pv_done"]
print("step " + " ".join(f"{n:>13s}" for n in names) + "   period(s_full)")
for j in range(1, 40):
    row = [ev[e][j] - t0 for e in range(8)]
    print(f"{j:4d} " + " ".join(f"{v:13d}" for v in row) + f"   {ev[4][j] - ev[4][j - 1]:6d}")

# the dQ pass (v10) of the same run: blockIdx (7, 0)
lib().mgv_dev_attn_trace(buf)
ev = [[buf[e * 64 + j] for j in range(64)] for e in range(8)]
t0 = ev[3][0]
names = ["mma:S(j) iss", "mma:dQ(j) iss", "mma:dP(j) iss", "cmp:s_full", "cmp:s_empty>", "cmp:exp done", "cmp:dp_full",
         "cmp:ds_full>"]
print("dQ pass")
print("step " + " ".join(f"{n:>13s}" for n in names) + "   period(s_full)")
for j in range(1, 40):
    row = [ev[e][j] - t0 for e in range(8)]
    print(f"{j:4d} " + " ".join(f"{v:13d}" for v in row) + f"   {ev[3][j] - ev[3][j - 1]:6d}")
