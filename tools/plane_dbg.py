import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from dpm_inputs.rng import random_boxes
from paper_1811_03557_b200 import api
n, dt = 128, float(sys.argv[1])
c = api.DPM(n, -1.1, 1.1, "sphere", (0, 0, 0), (1, 1, 1), 2, dt, "cauchy")
q = random_boxes(135, 1, n)
u = c.aux_solve_batch(torch.from_numpy(q).cuda()).cpu().numpy()[0]
np.save(f'/root/repo/gpurun_out/u_plane{os.environ.get("DPM_PLANE","1")}_{sys.argv[1]}.npy', u)
