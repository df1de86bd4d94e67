"""Summarise an ncu --set full report (first profiled kernel): key throughputs, stall reasons, opcode mix.

    python tools/ncu_summary.py report.ncu-rep
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]


def page(p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


rows = page("raw")
h, v = rows[0], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__inst_executed.sum"]
for name, val in zip(h, v):
    if name in want:
        print(f"{name:80s} {val}")
st = []
for name, val in zip(h, v):
    if "smsp__average_warps_issue_stalled" in name and name.endswith("per_issue_active.ratio"):
        try:
            st.append((float(val), name.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        except ValueError:
            pass
print("stalls (warps per issue):", ", ".join(f"{n}={x:.2f}" for x, n in sorted(st, reverse=True)[:8]))
rows = page("source", ("--print-source", "sass"))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hh = rows[hi]
isrc, iss, iex = hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
agg, ex, tot = defaultdict(float), defaultdict(float), 0.0
for r in rows[hi + 1:]:
    try:
        s, e = float(r[iss]), float(r[iex] or 0)
    except (ValueError, IndexError):
        continue
    op = [o for o in r[isrc].split() if not o.startswith("@")]
    k = op[0].split(".")[0] if op else "?"
    agg[k] += s
    ex[k] += e
    tot += s
print("opcode: stall-sample share / executed warp instructions")
for k, s in sorted(agg.items(), key=lambda x: -x[1])[:14]:
    print(f"  {k:8s} {s / tot * 100:5.1f}%  {ex[k]:.0f}")
