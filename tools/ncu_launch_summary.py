"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel name count,
total and mean duration (us), sorted by total."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
unit_i = h.index("Metric Unit") if "Metric Unit" in h else None
agg = defaultdict(lambda: [0, 0.0])
for r in rows[hdr + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    u = r[unit_i] if unit_i is not None else "ns"
    us = v / 1e3 if u in ("ns", "nsecond") else (v if u in ("us", "usecond") else v * 1e3)
    name = r[ki].split("(")[0][:56]
    if "Grid Size" in h:
        name += " g" + r[h.index("Grid Size")].replace(" ", "")
    agg[name][0] += 1
    agg[name][1] += us
tot = sum(a[1] for a in agg.values())
n = sum(a[0] for a in agg.values())
print(f"{n} launches, {tot/1e3:.3f} ms total kernel time")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:72s} n={c:6d} total={t/1e3:9.3f} ms mean={t/c:8.2f} us share={t/tot:5.3f}")
