"""Wall-time split of the cfg5 DD step (after the builds): python tools/dd_step_phases.py [steps]"""
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
for _ in range(12):   # past the 3 builds of the first steps
    sol.step()
torch.cuda.synchronize()
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
acc = {}
orig = {}
for name in ("local_begin", "local_finish_async", "stats", "cfl_async", "cfl_result"):
    orig[name] = getattr(api.Octant, name)

    def wrap(f, nm):
        def g(self, *a, **k):
            t0 = time.perf_counter()
            r = f(self, *a, **k)
            acc[nm] = acc.get(nm, 0.0) + time.perf_counter() - t0
            return r
        return g
    setattr(api.Octant, name, wrap(orig[name], name))
t0 = time.perf_counter()
for _ in range(steps):
    sol.step()
torch.cuda.synchronize()
tot = time.perf_counter() - t0
print(f"{1e3 * tot / steps:.3f} ms/step; host time inside octant calls per step (ms):",
      {k: round(1e3 * v / steps, 3) for k, v in acc.items()})
