"""Summarise an `ncu --page source --csv --print-source sass` export: mbarrier waits and hot lines.
usage: python tools/sass_hot.py export.csv [kernel-substring]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], None, []]
        blocks.append(cur)
    elif r and r[0] == "Address":
        cur[1] = r
    elif cur is not None and cur[1] is not None:
        cur[2].append(r)
for name, hdr, data in blocks:
    if want not in name:
        continue
    si, wi, ei = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    val = lambda r, i: int(r[i]) if r[i].strip() else 0
    tot = sum(val(r, wi) for r in data)
    print(name[:80], "samples", tot)
    for i, r in enumerate(data):
        if "TRYWAIT" in r[si] and i + 1 < len(data):
            n = data[i + 1]
            print(f"  {i:5d} exec={r[ei]:>8s} {r[si].strip()[:70]:70s} next={val(n, wi):6d} ({val(n, wi) / tot * 100:4.1f}%)")
    print("  hottest:")
    for i in sorted(range(len(data)), key=lambda i: -val(data[i], wi))[:12]:
        print(f"  {i:5d} {val(data[i], wi) / tot * 100:5.1f}%  {data[i][si].strip()[:80]}")
    break
