"""Test B steps (N = 127, 150 zonal harmonics) after a warm-up, at the initial dt (no rebuilds), for ncu launch
lists:  python tools/testb_launches.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from dpm_inputs import test_b_config  # noqa: E402
from paper_1811_03557_b200 import api  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cfg = test_b_config(127, 150)
ctx = api.DPM.from_config(cfg)
rho = torch.zeros((cfg.n,) * 3, dtype=torch.float64, device="cuda")
c = torch.zeros_like(rho)
ctx.pks_init(rho, c, cfg.ic_center, *cfg.ic_rho, *cfg.ic_c, rho_cell_average=True)
ctx.pks_step(rho, c, 10, chi=cfg.chi, dt_cap=cfg.dt)        # build + graph capture
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ctx.pks_step(rho, c, steps, chi=cfg.chi, dt_cap=cfg.dt)
e1.record()
e1.synchronize()
print(f"testB127: {e0.elapsed_time(e1) / steps * 1e3:.1f} us per step over {steps} steps")
