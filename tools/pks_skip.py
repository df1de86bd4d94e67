"""In-graph cost of each part of a PKS step: steps/s with DPM_STEP_SKIP=<mask> (parts left out of the
captured step graph; results wrong, timing only).  Needs a library built with the skip switches:
    DPM_NVCC_EXTRA=-DDPM_TIMING_SKIPS=1 python -m paper_1811_03557_b200.build --force
    python tools/pks_skip.py cfg3"""
import os
import subprocess
import sys

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
code = f"""
import sys, torch
sys.path.insert(0, '.')
from dpm_inputs import get_config
from paper_1811_03557_b200 import api
cfg = get_config('{cfg}')
ctx = api.DPM.from_config(cfg)
rho = torch.zeros((cfg.n,) * 3, dtype=torch.float64, device='cuda'); c = torch.zeros_like(rho)
ctx.pks_init(rho, c, cfg.ic_center, *cfg.ic_rho, *cfg.ic_c)
ctx.pks_step(rho, c, 10, chi=cfg.chi, dt_cap=cfg.dt)
ts = []
for r in range(7):
    ctx.pks_init(rho, c, cfg.ic_center, *cfg.ic_rho, *cfg.ic_c)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ctx.pks_step(rho, c, 100, chi=cfg.chi, dt_cap=cfg.dt); e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1) / 100 * 1e3)
ts.sort(); print(ts[3])
"""
for name, env in [("all", {}), ("-particular AP", {"DPM_STEP_SKIP": "1"}), ("-green AP", {"DPM_STEP_SKIP": "2"}),
                  ("-both AP", {"DPM_STEP_SKIP": "3"}), ("-trace/lsq/ext", {"DPM_STEP_SKIP": "4"}),
                  ("-green rhs", {"DPM_STEP_SKIP": "8"}), ("-restrict", {"DPM_STEP_SKIP": "16"}),
                  ("-resid", {"DPM_STEP_RESID": "0"}), ("only flux", {"DPM_STEP_SKIP": "31", "DPM_STEP_RESID": "0"}),
                  ("-x passes", {"DPM_SKIP_XPASS": "1"}), ("-plane", {"DPM_SKIP_PLANE": "1"})]:
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True)
    out = r.stdout.strip().splitlines()
    print(f"{cfg} {name:16s} {out[-1] if out else 'failed: ' + r.stderr[-300:]} us/step", flush=True)
