"""Config 5 (8-octant DD, R24) on one GPU: build + steps, timings and the dt / mass trajectory
(compare with SURVEY probe P12: dt 5.1174e-7 -> 8.4348e-8, 3 BEP builds, max rho 4.5247e4,
mass 6.0216302845 -> +344%)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from dpm_inputs import get_config
from paper_1811_03557_b200 import api
from paper_1811_03557_b200.dd import DDSolver

cfg = get_config("cfg5")
steps = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.steps
t0 = time.perf_counter()
octs = [api.Octant(cfg.n, cfg.lo, cfg.hi, s, 1.0, cfg.lmax, cfg.deg_if, cfg.dt) for s in range(8)]
torch.cuda.synchronize()
t_create = time.perf_counter() - t0
sol = DDSolver(octs, cfg.dt, chi=cfg.chi)
sol.init(cfg.ic_center, cfg.ic_rho, cfg.ic_c)
logs, t_build = [], 0.0
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(steps):
    b0 = sol.builds
    ts = time.perf_counter()
    logs.append(sol.step())
    torch.cuda.synchronize()
    if sol.builds > b0:
        t_build += time.perf_counter() - ts
t_tot = time.perf_counter() - t0
out = {"octants": 8, "n": cfg.n, "K": octs[0].K, "rows_per_octant": octs[0].n_rows, "steps": steps,
       "create_s": t_create, "total_s": t_tot, "build_s_incl_step": t_build, "builds": sol.builds,
       "steps_per_s_excl_builds": (steps - sol.builds) / max(t_tot - t_build, 1e-9),
       "dt_first": logs[0]["dt"], "dt_last": logs[-1]["dt"], "t_end": logs[-1]["t"],
       "mass_first": logs[0]["mass"], "mass_last": logs[-1]["mass"], "rho_max_last": logs[-1]["rho_max"],
       "rho_min_last": logs[-1]["rho_min"]}
print(json.dumps(out))
