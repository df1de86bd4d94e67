"""Per-phase durations of the FACR plane kernel from its optional clock64 instrumentation.

    DPM_NVCC_EXTRA="-DFACR_PHASE_TIMING=1" python -c "from paper_1811_03557_b200 import build as B; B.build(force=True)"
    python tools/facr_phases.py          # 16 fields at n = 128 = 4096 CTAs, all recorded
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from dpm_inputs.rng import random_boxes  # noqa: E402
from paper_1811_03557_b200 import api, _lib  # noqa: E402

n, nf = 128, 16
c = api.DPM(n, -1.1, 1.1, "sphere", (0, 0, 0), (1, 1, 1), 2, 1e-5, "cauchy")
q = torch.from_numpy(random_boxes(3, nf, n)).cuda()
for _ in range(3):
    c.aux_solve_batch(q)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (4096 * 9))()
rc = _lib.lib.dpm_debug_facr_phases(buf, 4096)
assert rc == 0, rc
t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 9).astype(np.int64)
d = np.diff(t, axis=1)
names = ["setup+load", "rhs (1)", "kept DST", "tri (3)", "kept iDST", "push/wait", "elim (5)", "store"]
ghz = float(sys.argv[1]) if len(sys.argv) > 1 else 1.965
tot = np.median(t[:, 8] - t[:, 0])
print(f"CTA lifetime median {tot:.0f} cycles = {tot / ghz / 1e3:.2f} us")
for r in (0, 1):
    dr = d[r::2]
    print(f"rank {r}: " + ", ".join(f"{nm} {np.median(dr[:, k]):.0f}" for k, nm in enumerate(names)))
print("share: " + ", ".join(f"{nm} {100 * np.median(d[:, k]) / tot:.0f}%" for k, nm in enumerate(names)))
