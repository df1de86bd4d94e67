"""Per-CUDA-source-line stall samples and shared-memory wavefronts from an ncu report
(--page source --print-source cuda,sass), optionally grouped into line ranges.

    python tools/ncu_lines.py report.ncu-rep [top] [name:lo-hi ...]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
iS, iW, iI = h.index("# Samples"), h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal")
lines = []
for r in rows[hi + 1:]:
    if r and r[0] and len(r) > iI:
        try:
            lines.append((int(r[iS]), int(r[0]), r[1][:80], int(r[iW] or 0), int(r[iI] or 0)))
        except ValueError:
            pass
tot = sum(x[0] for x in lines)
print("total samples", tot)
for s, l, src, w, idl in sorted(lines, reverse=True)[:top]:
    print(f"{s:7d} {100 * s / tot:5.1f}% L{l:4d} wf={w:10d} ideal={idl:10d} {src}")
for spec in sys.argv[3:]:
    name, rng = spec.split(":")
    lo, hi_ = map(int, rng.split("-"))
    s = sum(x[0] for x in lines if lo <= x[1] <= hi_)
    print(f"{name:12s} L{lo}-{hi_}: {100 * s / tot:5.1f}%")
