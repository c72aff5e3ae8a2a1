"""Per-kernel medians of an alternating A/B log (tools/ab_fusions_full.sh / tools/ab_libs_full.sh output):
    python tools/ab_table.py LOG [min_delta_ms]"""
import collections
import re
import statistics as st
import sys

runs, cur = [], None
for line in open(sys.argv[1]):
    m = re.match(r"== (?:fusions|lib) (\S+)", line)
    if m:
        cur = {"arm": m.group(1), "k": {}}
        runs.append(cur)
        continue
    m = re.match(r"total kernel time per step: ([\d.]+)", line)
    if m and cur is not None:
        cur["total"] = float(m.group(1))
        continue
    m = re.match(r"\s+([\d.]+) ms\s+[\d.]+% x\s*(\d+)\s+(.*)", line)
    if m and cur is not None:
        name = re.sub(r"\(.*", "", re.sub(r"\(CUtensorMap.*", "", m.group(3)))
        cur["k"][name] = cur["k"].get(name, 0.0) + float(m.group(1))
arms = list(dict.fromkeys(r["arm"] for r in runs))
for a in arms:
    t = [r["total"] for r in runs if r["arm"] == a and "total" in r]
    print(f"{a}: total kernel ms/step median {st.median(t):.2f}  runs {', '.join(f'{x:.2f}' for x in t)}")
if len(arms) == 2:
    A, B = arms
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in runs:
        for k, v in r["k"].items():
            agg[k][r["arm"]].append(v)
    thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.02
    rows = []
    for k, d in agg.items():
        a = st.median(d[A]) if d.get(A) else 0.0
        b = st.median(d[B]) if d.get(B) else 0.0
        if abs(a - b) > thr:
            rows.append((b - a, k, a, b))
    for dlt, k, a, b in sorted(rows):
        print(f"{dlt:+7.3f}  A:{a:8.3f} B:{b:8.3f}  {k[:100]}")
