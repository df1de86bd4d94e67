"""Run the cfg2 / cfg3 PKS loop once (for ncu launch lists)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from dpm_inputs import get_config
from paper_1811_03557_b200 import api

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = get_config(name)
ctx = api.DPM.from_config(cfg)
n = cfg.n
rho = torch.zeros((n, n, n), dtype=torch.float64, device="cuda")
c = torch.zeros_like(rho)
ctx.pks_init(rho, c, cfg.ic_center, *cfg.ic_rho, *cfg.ic_c)
ctx.pks_step(rho, c, cfg.steps, chi=cfg.chi, dt_cap=cfg.dt)
torch.cuda.synchronize()
ctx.pks_init(rho, c, cfg.ic_center, *cfg.ic_rho, *cfg.ic_c)
ctx.pks_step(rho, c, cfg.steps, chi=cfg.chi, dt_cap=cfg.dt)
torch.cuda.synchronize()
print("ok")
