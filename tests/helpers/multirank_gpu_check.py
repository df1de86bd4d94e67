"""Multi-rank GPU check, run under torch.distributed.run by tests/test_gpu_multirank.py.

Every rank uses cuda:0 and the collectives go over gloo (NCCL refuses two ranks on one device; the box has
one GPU).  The kernels of different ranks never wait on one another: only the host-side collectives couple
them.  Checked against the same work done by this rank alone:
  * C1: parallel.build_projection_distributed at the cfg3 geometry (columns sharded over the
    ranks, one all-gather, local CholeskyQR2) against ctx.build_projection(): B bit-identical, LSQ
    coefficients <= 1e-12;
  * cfg5-style DD at n = 16: the 8 octants sharded over the ranks (8/W each; W = 8 takes the per-octant
    dpm_dd_local_begin/finish path) against all 8 octants in one DDSolver on this rank: dt sequence
    <= 1e-12, rho and c of the rank's octants and the mass <= 1e-9 (R23) after 3 steps with a rebuild.
Rank 0 prints one JSON line with the measured differences.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from dpm_inputs import get_config  # noqa: E402
from paper_1811_03557_b200 import api, parallel  # noqa: E402
from paper_1811_03557_b200.dd import DDSolver  # noqa: E402

N, LC, LI, BOX = 16, 4, 4, (-0.1, 1.1)
IC_RHO, IC_C = (1000.0, 100.0), (500.0, 50.0)


def rel(a, b):
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-300))


def dd_run(octant_ids, use_dist, steps=3):
    octs = [api.Octant(N, *BOX, s, 1.0, LC, LI, 1e-3, device=0) for s in octant_ids]
    sol = DDSolver(octs, 1e-3, chi=1.0)
    if not use_dist:   # the single-process run must not enter the collectives of the group
        import paper_1811_03557_b200.dd as ddm
        saved, ddm._allreduce = ddm._allreduce, (lambda t, op: t)
    try:
        sol.init((0.0, 0.0, 0.0), IC_RHO, IC_C)
        logs = []
        for i in range(steps):
            if i == steps - 1:
                sol.dt_cap *= 0.5       # forces a Step-4b rebuild on the last step
            logs.append(sol.step())
        torch.cuda.synchronize()
    finally:
        if not use_dist:
            ddm._allreduce = saved
    return sol, logs


def main():
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    out = {"world": world}

    # ---- C1: distributed BEP build on the GPU
    cfg = get_config("cfg3")
    ctx = api.DPM.from_config(cfg, device=0)
    Bd = parallel.build_projection_distributed(ctx, world, rank)
    g = torch.from_numpy(np.random.default_rng(7).uniform(-1, 1, (2, ctx.info["n_gamma_in"]))).cuda()
    cd, _ = ctx.boundary_lsq(g)
    _, Bs = ctx.build_projection()
    cs, _ = ctx.boundary_lsq(g)
    out["bep_B_equal"] = bool(torch.equal(Bd, Bs))
    out["bep_coef_rel"] = rel(cd, cs)
    del ctx

    # ---- DD: octants sharded over the ranks vs all 8 on this rank
    per = 8 // world
    mine = list(range(rank * per, (rank + 1) * per))
    sol_d, logs_d = dd_run(mine, True)
    sol_s, logs_s = dd_run(list(range(8)), False)
    out["dd_path"] = "batched" if sol_d._batched() else "per-octant local_begin/finish"
    out["dd_builds"], out["dd_builds_single"] = sol_d.builds, sol_s.builds
    out["dd_dt_rel"] = max(abs(a["dt"] - b["dt"]) / b["dt"] for a, b in zip(logs_d, logs_s))
    out["dd_mass_rel"] = max(abs(a["mass"] - b["mass"]) / abs(b["mass"]) for a, b in zip(logs_d, logs_s))
    e = 0.0
    for i, s in enumerate(mine):
        for k in (0, 1):
            e = max(e, rel(sol_d.fields[i][k], sol_s.fields[s][k]))
    t = torch.tensor([e, out["dd_dt_rel"], out["dd_mass_rel"], out["bep_coef_rel"],
                      0.0 if out["bep_B_equal"] else 1.0], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out["dd_field_rel"], out["dd_dt_rel"], out["dd_mass_rel"], out["bep_coef_rel"] = (float(x) for x in t[:4])
    out["bep_B_equal"] = float(t[4]) == 0.0
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
