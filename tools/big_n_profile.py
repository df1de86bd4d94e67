"""Per-pass times of the AP solve at n in (128, 320] (the paper's N = 132 / 255 / 260 meshes):
batches of 2 fields (the PKS step's shape) and of 16, dpm_set_pass_timing split, vs HBM bytes.

    python tools/big_n_profile.py [n ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from dpm_inputs.rng import random_boxes  # noqa: E402
from paper_1811_03557_b200 import api  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [132, 255, 260]:
    c = api.DPM(n, -1.1, 1.1, "sphere", (0, 0, 0), (1, 1, 1), 0, 1e-5, "cauchy")
    for b in (2, 16):
        q = torch.from_numpy(random_boxes(1, b, n)).cuda()
        u = torch.empty_like(q)
        for _ in range(3):
            c.aux_solve_batch(q, u)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            c.aux_solve_batch(q, u)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        c.set_pass_timing(True)
        c.aux_solve_batch(q, u)
        torch.cuda.synchronize()
        pt = c.pass_times()
        c.set_pass_timing(False)
        byts = 16.0 * n ** 3 * b
        print(json.dumps({"n": n, "batch": b, "ms": ms, "solves_per_s": b / ms * 1e3,
                          "one_pass_TBs": byts / ms / 1e9, "passes": pt}))
