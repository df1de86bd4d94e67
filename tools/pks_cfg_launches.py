"""PKS steps of config 2 or 3 after a warm-up (for ncu launch lists / --set full captures of the step's
kernels):  python tools/pks_cfg_launches.py cfg3 10"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from dpm_inputs import get_config  # noqa: E402
from paper_1811_03557_b200 import api  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = get_config(name)
ctx = api.DPM.from_config(cfg)
rho = torch.zeros((cfg.n,) * 3, dtype=torch.float64, device="cuda")
c = torch.zeros_like(rho)
ctx.pks_init(rho, c, cfg.ic_center, *cfg.ic_rho, *cfg.ic_c)
ctx.pks_step(rho, c, 10, chi=cfg.chi, dt_cap=cfg.dt)        # build + graph capture
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ctx.pks_step(rho, c, steps, chi=cfg.chi, dt_cap=cfg.dt)
e1.record()
e1.synchronize()
print(f"{name}: {e0.elapsed_time(e1) / steps * 1e3:.1f} us per step over {steps} steps")
