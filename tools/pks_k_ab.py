import sys, torch, statistics
sys.path.insert(0, '.')
from dpm_inputs import get_config
from paper_1811_03557_b200 import api
for name, steps in (("cfg2", 100), ("cfg3", 100), ("cfg2", 10)):
    cfg = get_config(name)
    ctx = api.DPM.from_config(cfg)
    rho = torch.zeros((cfg.n,) * 3, dtype=torch.float64, device='cuda'); c = torch.zeros_like(rho)
    ctx.pks_init(rho, c, cfg.ic_center, *cfg.ic_rho, *cfg.ic_c)
    ctx.pks_step(rho, c, steps, chi=cfg.chi, dt_cap=cfg.dt)
    ts = []
    for r in range(9):
        ctx.pks_init(rho, c, cfg.ic_center, *cfg.ic_rho, *cfg.ic_c)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); ctx.pks_step(rho, c, steps, chi=cfg.chi, dt_cap=cfg.dt); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1) / steps * 1e3)
    print(name, steps, round(statistics.median(ts), 2), "us/step")
