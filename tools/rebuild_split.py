import sys, time, torch
sys.path.insert(0, '.')
from dpm_inputs import get_config
from paper_1811_03557_b200 import api
cfg = get_config("cfg3")
ctx = api.DPM.from_config(cfg)
n = cfg.n
rho = torch.zeros((n,)*3, dtype=torch.float64, device="cuda"); c = torch.zeros_like(rho)
ctx.pks_init(rho, c, cfg.ic_center, *cfg.ic_rho, *cfg.ic_c)
dt0 = ctx.pks_step(rho, c, 1, chi=cfg.chi, dt_cap=cfg.dt)[0]["dt"]
ctx.pks_step(rho, c, 2, chi=cfg.chi, dt_cap=dt0*0.999, dt_rule=1)
torch.cuda.synchronize()
# 1) whole loop
t0 = time.perf_counter()
for i in range(20):
    ctx.pks_step(rho, c, 1, chi=cfg.chi, dt_cap=dt0*(1-1e-3*(i+2)), dt_rule=1)
torch.cuda.synchronize(); print("rebuild+step %.3f ms" % ((time.perf_counter()-t0)/20*1e3))
# 2) build_projection alone at new dts
t0 = time.perf_counter()
for i in range(20):
    ctx.set_dt(dt0*(1-1e-3*(i+40)))
    ctx.build_projection(False)
torch.cuda.synchronize(); print("build_projection %.3f ms" % ((time.perf_counter()-t0)/20*1e3))
# 3) bep columns alone
t0 = time.perf_counter()
for i in range(20):
    ctx.bep_columns(0, ctx.K)
torch.cuda.synchronize(); print("bep_columns %.3f ms" % ((time.perf_counter()-t0)/20*1e3))
# 4) step at a fixed (cached) dt
dtf = dt0*(1-1e-3*60)
ctx.pks_step(rho, c, 1, chi=cfg.chi, dt_cap=dtf, dt_rule=1)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(20):
    ctx.pks_step(rho, c, 1, chi=cfg.chi, dt_cap=dtf, dt_rule=1)
torch.cuda.synchronize(); print("single cached step call %.3f ms" % ((time.perf_counter()-t0)/20*1e3))
