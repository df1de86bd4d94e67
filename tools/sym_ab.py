"""NEXT-1 octant path (bep_sym.cu) A/B: dpm_bep_columns over all K columns of cfg1-cfg4 (median of 5, CUDA
events) in this process's mode (DPM_BEP_SYM unset / 0 / 2), the columns saved for comparison."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from dpm_inputs import get_config  # noqa: E402
from paper_1811_03557_b200 import api  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else None
res = {}
for name in os.environ.get("SYM_CFGS", "cfg1,cfg2,cfg3,cfg4").split(","):
    ctx = api.DPM.from_config(get_config(name))
    K = ctx.K
    PgE, B = ctx.bep_columns(0, K)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.bep_columns(0, K)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    ctx.build_projection(want_outputs=False)
    tb = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.build_projection(want_outputs=False)
        e1.record()
        e1.synchronize()
        tb.append(e0.elapsed_time(e1))
    # one boundary LSQ on a fixed random right-hand side (coefficients compared across modes)
    g = torch.from_numpy(np.random.default_rng(7).uniform(-1, 1, (1, ctx.info["n_gamma_in"]))).cuda()
    coef, ug = ctx.boundary_lsq(g)
    res[name] = {"K": K, "columns_ms": ms, "columns_per_s": K / ms * 1e3, "build_ms": statistics.median(tb)}
    if out:
        np.save(f"{out}_{name}_coef.npy", coef.cpu().numpy())
        np.save(f"{out}_{name}_ug.npy", ug.cpu().numpy())
    if out:
        np.save(f"{out}_{name}_pg.npy", PgE.cpu().numpy())
        np.save(f"{out}_{name}_b.npy", B.cpu().numpy())
    del ctx
print(json.dumps({"sym": os.environ.get("DPM_BEP_SYM", "1"), **res}))
