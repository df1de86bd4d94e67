"""A few PKS steps of the paper's Test B at mesh N (default 255) for a launch list:

    ncu --metrics gpu__time_duration.sum --csv --log-file out.csv python tools/pks_step_launches.py 255 3
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from dpm_inputs import test_b_config  # noqa: E402
from paper_1811_03557_b200 import api  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 255
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = test_b_config(N, 300 if N > 200 else 150)
ctx = api.DPM.from_config(cfg)
rho = torch.zeros((cfg.n,) * 3, dtype=torch.float64, device="cuda")
c = torch.zeros_like(rho)
ctx.pks_init(rho, c, cfg.ic_center, *cfg.ic_rho, *cfg.ic_c)
ctx.pks_step(rho, c, 1, chi=cfg.chi, dt_cap=cfg.dt, dt_rule=0, clamp=1)   # build + first step
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ctx.pks_step(rho, c, steps, chi=cfg.chi, dt_cap=cfg.dt, dt_rule=0, clamp=1)
e1.record()
e1.synchronize()
print(f"N={N}: {e0.elapsed_time(e1) / steps:.3f} ms per step over {steps} steps")
