"""Timeline of one dK/dV CTA pair from a -DMGV_ATTN_TRACE build (variants/trace)."""
import ctypes
import os
import sys

os.environ["MGV_LIB_PATH"] = "variants/trace/libmugv_b200.so"
sys.argv = ["probe", os.environ.get("TN", "14400"), "none", "1"]
exec(open("tools/probe_attn.py").read())  # builds the inputs and runs the forward once
dO = (torch.randn(N, H, device="cuda", generator=g) * 0.1).bfloat16()
Dv = torch.empty(heads, (N + 63) // 64 * 64, device="cuda")
dqkv = torch.empty(N, 3 * H, device="cuda").bfloat16()
L.mgv_dev_attn_bwd(1, P(qkv.data_ptr()), i64(3 * H), P(qkv[:, H:].data_ptr()), i64(3 * H),
                   P(qkv[:, 2 * H:].data_ptr()), i64(3 * H), P(o.data_ptr()), i64(H), P(lse.data_ptr()),
                   P(dO.data_ptr()), i64(H), P(Dv.data_ptr()), P(dqkv.data_ptr()), i64(3 * H),
                   P(dqkv[:, H:].data_ptr()), i64(3 * H), P(dqkv[:, 2 * H:].data_ptr()), i64(3 * H),
                   P(0), 1, N, N, heads, hd, P(stream))
torch.cuda.synchronize()
from paper_2510_17519_b200._lib import lib  # noqa: E402
buf = (ctypes.c_ulonglong * (8 * 64))()
lib().mgv_dev_attn_trace2(buf)
ev = [[buf[e * 64 + j] for j in range(64)] for e in range(8)]
names = ["S/dP ok", "TMEM st ok", "xfree ok", "sent"]
for r in range(2):
    t0 = ev[4 * r][0]
    print(f"CTA {r}: step " + " ".join(f"{n:>11s}" for n in names) + "   period")
    for j in range(1, 24):
        row = [ev[4 * r + e][j] - t0 for e in range(4)]
        print(f"      {j:4d} " + " ".join(f"{v:11d}" for v in row) + f"   {ev[4 * r][j] - ev[4 * r][j - 1]:6d}")
