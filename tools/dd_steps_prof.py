"""cfg5 DD steady-state steps for ncu (--profile-from-start off): 12 warm steps (3 builds), then 5 profiled."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from dpm_inputs import get_config  # noqa: E402
from paper_1811_03557_b200 import api  # noqa: E402
from paper_1811_03557_b200.dd import DDSolver  # noqa: E402

cfg = get_config("cfg5")
octs = [api.Octant(cfg.n, cfg.lo, cfg.hi, s, 1.0, cfg.lmax, cfg.deg_if, cfg.dt) for s in range(8)]
sol = DDSolver(octs, cfg.dt, chi=cfg.chi)
sol.init(cfg.ic_center, cfg.ic_rho, cfg.ic_c)
for _ in range(12):
    sol.step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(5):
    sol.step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
