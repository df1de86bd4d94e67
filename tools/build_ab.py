"""BEP build latency at cfg1 (K = 50), cfg3 (K = 242) and cfg4 (K = 578): dpm_build_projection, median of
reps, CUDA events (factorisation + columns)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from dpm_inputs import get_config  # noqa: E402
from paper_1811_03557_b200 import api  # noqa: E402

out = {}
for name in ("cfg1", "cfg3", "cfg4"):
    ctx = api.DPM.from_config(get_config(name))
    ctx.build_projection(False)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.build_projection(False)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    out[name] = statistics.median(ts)
print(json.dumps({"build_projection_ms": out}))
