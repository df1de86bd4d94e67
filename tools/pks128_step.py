import sys, time, torch
sys.path.insert(0, '.')
from dpm_inputs import get_config
from paper_1811_03557_b200 import api
cfg = get_config("cfg4")   # n = 128 sphere geometry, K = 578
ctx = api.DPM.from_config(cfg)
n = cfg.n
rho = torch.zeros((n,)*3, dtype=torch.float64, device="cuda"); c = torch.zeros_like(rho)
ctx.pks_init(rho, c, (0.0, 0.0, 0.0), 1000.0, 100.0, 500.0, 50.0)
ctx.pks_step(rho, c, 10, chi=1.0, dt_cap=1e-6, dt_rule=1)
torch.cuda.synchronize()
t0 = time.perf_counter()
ctx.pks_step(rho, c, 100, chi=1.0, dt_cap=1e-6, dt_rule=1)
torch.cuda.synchronize()
print("n=128 K=578 PKS step %.1f us" % ((time.perf_counter() - t0) / 100 * 1e6))
