"""cfg5 DD steps/s (bench.py's bench_dd, 3 repeats of the 50-step loop): A/B of DPM_DD_SHARED."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1811_03557_b200 import api  # noqa: E402

r = bench.bench_dd(api, torch, 1, 0, reps=3)
print(json.dumps({"shared": os.environ.get("DPM_DD_SHARED", "1"), "steps_per_s": r["steps_per_s_excl_builds"],
                  "builds": r["builds"], "dt_last": r["dt_last"], "mass_end": r["mass_end"], "rho_max_end": r["rho_max_end"]}))
