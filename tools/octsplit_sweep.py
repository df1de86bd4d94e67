"""2-field AP solve time (CUDA events, 50 solves) over n in (64, 128): parity-split solver vs the generic passes.
    python tools/octsplit_sweep.py     # runs itself with DPM_OCTSPLIT=2 (every n) / 0
"""
import dataclasses
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
NS = [65, 68, 72, 80, 88, 96, 100, 104, 112, 120, 126, 127]


def one():
    import torch
    from dpm_inputs import get_config
    from paper_1811_03557_b200 import api
    out = {}
    for n in NS:
        cfg = dataclasses.replace(get_config("cfg1"), n=n, lmax=1)
        ctx = api.DPM.from_config(cfg)
        q = torch.rand((2, n, n, n), dtype=torch.float64, device="cuda")
        u = torch.empty_like(q)
        for _ in range(3):
            ctx.aux_solve_batch(q, u)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            ctx.aux_solve_batch(q, u)
        e1.record()
        e1.synchronize()
        out[n] = round(e0.elapsed_time(e1) / 50 * 1e3, 1)
        del ctx
    print(os.environ.get("DPM_OCTSPLIT", "1"), json.dumps(out), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        one()
    else:
        for v in ("2", "0"):
            subprocess.run([sys.executable, os.path.abspath(__file__), "one"], env=dict(os.environ, DPM_OCTSPLIT=v))
