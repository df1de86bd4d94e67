"""Summarise an ncu --csv launch list with one or more metrics: per kernel count, mean duration, mean DRAM
bytes read / written (when captured)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = defaultdict(dict)
names = {}
for r in rows[hdr + 1:]:
    if len(r) > vi:
        d[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = r[ki].split("(")[0][:50]
agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i, m in d.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0)
    a[3] += m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:50s} n={a[0]:4d} avg={a[1] / a[0] / 1e3:9.1f} us share={a[1] / tot:6.1%} "
          f"rd={a[2] / a[0] / 1e6:8.1f} MB wr={a[3] / a[0] / 1e6:8.1f} MB")
