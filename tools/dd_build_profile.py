"""One config-5 octant BEP build + factorisation (for ncu launch lists)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from dpm_inputs import get_config
from paper_1811_03557_b200 import api
from paper_1811_03557_b200.dd import DDSolver
cfg = get_config("cfg5")
nocts = int(sys.argv[1]) if len(sys.argv) > 1 else 2
octs = [api.Octant(cfg.n, cfg.lo, cfg.hi, s, 1.0, cfg.lmax, cfg.deg_if, 5e-7) for s in range(nocts)]
sol = DDSolver(octs, cfg.dt)
sol.build(5e-7)
torch.cuda.synchronize()
print("ok")
