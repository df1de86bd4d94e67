"""In-step cost of the parts of a cfg5 DD step (8 octants on one GPU): the DDSolver step with one Octant
phase replaced by a no-op (results wrong, timing only; the per-octant streams and syncs stay).
    python tools/dd_skip.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from dpm_inputs import get_config  # noqa: E402
from paper_1811_03557_b200 import api  # noqa: E402
from paper_1811_03557_b200.dd import DDSolver  # noqa: E402

cfg = get_config("cfg5")
octs = [api.Octant(cfg.n, cfg.lo, cfg.hi, s, 1.0, cfg.lmax, cfg.deg_if, cfg.dt) for s in range(8)]
sol = DDSolver(octs, cfg.dt, chi=cfg.chi)
sol.init(cfg.ic_center, cfg.ic_rho, cfg.ic_c)
for _ in range(12):   # past the builds
    sol.step()
torch.cuda.synchronize()
dt_fixed = sol.dt_prev


def timed(steps=30):
    sol.dt_rule = 1          # fixed dt: no CFL round trip changes, no rebuilds
    sol.dt_cap = dt_fixed
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        sol.step()
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0) / steps


def noop_y(self, *a, **k):
    return torch.zeros((2, self.K), dtype=torch.float64, device=self.device)


print(f"all (fixed dt)     {timed():.3f} ms/step", flush=True)
for name, repl in (("dd_rhs", lambda self, *a, **k: None), ("dd_green_rhs", lambda self, *a, **k: None),
                   ("dd_restrict", lambda self, *a, **k: None), ("dd_lsq_rhs_shared", lambda self, octs, *a, **k: noop_y(self)),
                   ("aux_solve_batch", lambda self, *a, **k: None)):
    orig = getattr(api.Octant, name, None) or getattr(api.DPM, name)
    setattr(api.Octant, name, repl)
    try:
        print(f"- {name:18s} {timed():.3f} ms/step", flush=True)
    except Exception as e:   # noqa: BLE001
        print(f"- {name:18s} failed: {str(e)[:80]}", flush=True)
    setattr(api.Octant, name, orig)
