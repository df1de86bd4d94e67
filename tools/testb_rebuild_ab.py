"""Step-4b rebuild at the paper's Test B mesh (N = 127, odd n, 150 zonal harmonics): build_projection and
bep_columns timings and the whole Test B run, octant path (default) vs DPM_BEP_SYM=0 (full grid).

    python tools/testb_rebuild_ab.py            # runs itself once per setting
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one():
    import torch
    from dpm_inputs import test_b_config
    from paper_1811_03557_b200 import api
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import test_b
    cfg = test_b_config(127, 150)
    ctx = api.DPM.from_config(cfg)
    out = {"sym": os.environ.get("DPM_BEP_SYM", "1"), "K": ctx.K}
    for name, fn in (("build_projection_ms", lambda i: (ctx.set_dt(cfg.dt * (1 - 1e-3 * (i + 1))), ctx.build_projection(False))),
                     ("bep_columns_ms", lambda i: ctx.bep_columns(0, ctx.K))):
        fn(0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(10):
            fn(i + 1)
        e1.record()
        e1.synchronize()
        out[name] = e0.elapsed_time(e1) / 10
    del ctx
    test_b.run(127, 150)
    res, _ = test_b.run(127, 150)
    out.update({k: res[k] for k in ("wall_s", "steps", "rebuilds", "t_stop", "steps_per_s")})
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        one()
    else:
        for sym in ("1", "0"):
            subprocess.run([sys.executable, os.path.abspath(__file__), "one"], env=dict(os.environ, DPM_BEP_SYM=sym))
