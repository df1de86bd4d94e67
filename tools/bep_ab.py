"""NEXT-1 A/B: dpm_bep_columns over the 578 columns of the cfg4 geometry (median of reps, CUDA events),
and the columns themselves against the dense-path columns (DPM_BEP_FUSED=0 run in-process is not possible:
the comparison is against a stored run, see tests)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from dpm_inputs import get_config  # noqa: E402
from paper_1811_03557_b200 import api  # noqa: E402

ctx = api.DPM.from_config(get_config("cfg4"))
K = ctx.K
ctx.bep_columns(0, K)
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.bep_columns(0, K)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = statistics.median(ts)
print(json.dumps({"columns_ms": ms, "columns_per_s": K / ms * 1e3, "zbox": os.environ.get("DPM_BEP_ZBOX", "1")}))
