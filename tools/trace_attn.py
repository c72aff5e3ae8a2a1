"""Timeline of one dQ CTA from a -DMGV_ATTN_TRACE build (variants/trace): per-step event clocks."""
import ctypes
import os
import subprocess
import sys

os.environ["MGV_LIB_PATH"] = "variants/trace/libmugv_b200.so"
sys.argv = ["probe", "14400", "bwd", "1"]
exec(open("tools/probe_attn.py").read())
from paper_2510_17519_b200._lib import lib  # noqa: E402
buf = (ctypes.c_ulonglong * (8 * 64))()
lib().mgv_dev_attn_trace(buf)
ev = [[buf[e * 64 + j] for j in range(64)] for e in range(8)]
t0 = ev[3][0]
names = ["mma:S(j+2)", "mma:dpE(j)", "mma:dsF(j)", "cmp:S(j+1) ok", "cmp:dP ok", "cmp:math done", "cmp:dsF arrive"]
print("step " + " ".join(f"{n:>14s}" for n in names) + "   period")
for j in range(2, 40):
    row = [ev[e][j] - t0 for e in range(7)]
    print(f"{j:4d} " + " ".join(f"{v:14d}" for v in row) + f"   {ev[3][j] - ev[3][j - 1]:6d}")
