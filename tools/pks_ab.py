"""PKS steps/s for cfg2 / cfg3 (bench.py's bench_pks: median of 20 repeats of the step loop) — used for
A/B runs of launch-path changes (e.g. DPM_PDL=0 vs 1)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1811_03557_b200 import api  # noqa: E402

out = {name: bench.bench_pks(api, torch, name) for name in ("cfg2", "cfg3")}
print(json.dumps({k: {"steps_per_s": v["steps_per_s"], "ms_per_step": v["ms_per_step"]} for k, v in out.items()}))
