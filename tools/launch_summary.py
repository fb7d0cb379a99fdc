"""Per-kernel totals of the LAST solve in an ncu launch-list CSV.

    python tools/launch_summary.py LIST.csv SOLVES
"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
solves = int(sys.argv[2]) if len(sys.argv) > 2 else 1
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
launches = []
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    unit = r[ui]
    ms = v / 1e6 if unit in ("nsecond", "ns") else v / 1e3 if unit in ("usecond", "us") else v
    launches.append((r[ki].split("(")[0].split("<")[0][-40:], ms))
per = len(launches) // solves
last = launches[-per:]
agg = OrderedDict()
for k, ms in last:
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += ms
tot = sum(v[1] for v in agg.values())
print(f"{len(last)} launches, {tot:.3f} ms kernel time in the last solve")
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {ms:8.3f} ms  {n:4d}x  {k}")
