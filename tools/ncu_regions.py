"""Stall samples of an ncu report by SASS region (windows of W instructions), with the stall reasons that
matter and the dominant opcodes of each window: where along the kernel the warps wait, and for what.

    python tools/ncu_regions.py report.ncu-rep [W]
"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
W = int(sys.argv[2]) if len(sys.argv) > 2 else 250
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h, data = rows[hi], rows[hi + 1:]
ix = {n: i for i, n in enumerate(h)}
val = lambda r, k: int(r[ix[k]] or 0)   # noqa: E731
stalls = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
total = sum(val(r, "# Samples") for r in data)
tot = {s: sum(val(r, s) for r in data) for s in stalls}
print(rows[0][1])
print("samples", total, "| SASS instructions", len(data))
print("stall share of all samples:", ", ".join(f"{k[6:]} {100 * v / total:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:10]))
cols = ["stall_no_inst", "stall_wait", "stall_long_sb", "stall_short_sb", "stall_barrier", "stall_math"]
print(f"{'instr':>6} {'samples':>8} " + " ".join(f"{c[6:]:>9}" for c in cols) + f" {'executed':>9}  top opcodes")
for i in range(0, len(data), W):
    seg = data[i:i + W]
    s = sum(val(r, "# Samples") for r in seg)
    if not s:
        continue
    ops = {}
    for r in seg:
        m = re.match(r"\s*(@!?U?P\d+\s+)?([A-Z0-9_.]+)", r[1])
        if m:
            o = m.group(2).split(".")[0]
            ops[o] = ops.get(o, 0) + 1
    top = " ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:3])
    print(f"{i:6d} {100 * s / total:7.1f}% " + " ".join(f"{100 * sum(val(r, c) for r in seg) / total:8.1f}%" for c in cols)
          + f" {sum(val(r, 'Instructions Executed') for r in seg) / 1e6:8.1f}M  {top}")
