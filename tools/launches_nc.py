"""Print a multi-metric ncu --csv launch list (one row per launch): id, kernel, duration, DRAM/L2 bytes."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = OrderedDict()
for r in rows[hi + 1:]:
    d.setdefault((r[ii], r[ki].split("(")[0][:44]), {})[r[mi]] = float(r[vi].replace(",", ""))
print(f"{'id':>3} {'kernel':44s} {'us':>8} {'dramR MB':>9} {'dramW MB':>9} {'L2 MB':>8}")
for (i, k), m in d.items():
    print(f"{i:>3} {k:44s} {m.get('gpu__time_duration.sum', 0) / 1e3:8.1f} {m.get('dram__bytes_read.sum', 0) / 1e6:9.1f} "
          f"{m.get('dram__bytes_write.sum', 0) / 1e6:9.1f} {m.get('lts__t_bytes.sum', 0) / 1e6:8.1f}")
