"""NEXT-3: the paper's two-subdomain domain decomposition (Case 1) on Test A — the DD
columns of Tables 1-3 and a B200 analogue of Table 6's R_S, on one GPU.

Tables 1-3: DD runs on the paper's "N1/N2" meshes (h_l = 2 r_l / (N_l - 4), r1 = 0.25, r2 = 0.5,
P:596) with Test A's IC (ρ̄0 as cell averages, R36/R38), one zonal harmonic per term on Z
and Γ, fixed Δt = 1e-8 to T = 1e-6, against the paper's reference, the SD run on N = 516:
* E∞ per subdomain (eq. dd-error-in-max-norm): max over M_l+ of |ρ̄_l - ρ̄*| at T, the
  reference restricted to each coarse cell [x ± h_l/2]^3 by the mean of the (h_l/h*)^3 fine values inside
  it (R37; the cells of every N_l/r_l mesh are unions of N = 516 cells);
* E_rel (eq. dd-conv-max-density-in-space) of max_l ||ρ̄_l||∞ over M_l+ (eq. dd-norm:max) per step.
Table 6: wall-clock of the SD run on N and of the DD runs N1/N2 to T = 6e-5 with Δt = min(0.5 h²,
CFL) (R13; the DD takes the minimum over both subdomains), BEP builds included; R_S = T_SD/T_DD
(P:931).  The paper's R_S were measured on a 32-core CPU node: context only.

    python tools/test_a_dd.py [--tables] [--rs]
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from dpm_inputs import paper_mesh, test_a_config  # noqa: E402
from paper_1811_03557_b200 import api  # noqa: E402
from paper_1811_03557_b200.dd import DDSolver  # noqa: E402

R1, R2 = 0.25, 0.5
# (N1, N2): (E∞ρ Ω1, E∞ρ Ω2, E∞c Ω1, E∞c Ω2, E_rel) — Table 1, Table 2, Table 3
PAPER_DD = {
    (20, 20): (1.4046e+00, 3.5954e-02, 5.6759e+00, 1.0804e+00, 1.0196e-01),
    (36, 36): (3.6990e-01, 8.3515e-03, 1.4766e+00, 2.8497e-01, 2.6378e-02),
    (68, 68): (1.2224e-01, 2.6776e-03, 3.5615e-01, 7.1525e-02, 6.3461e-03),
    (132, 132): (2.7815e-02, 7.7097e-04, 7.1459e-02, 1.7233e-02, 1.2724e-03),
    (20, 12): (1.4046e+00, 1.1226e-01, 5.6759e+00, 3.4957e+00, 1.0196e-01),
    (36, 20): (3.6990e-01, 3.7364e-02, 1.4766e+00, 1.0809e+00, 2.6378e-02),
    (68, 36): (1.2224e-01, 1.0093e-02, 3.5615e-01, 2.8524e-01, 6.3461e-03),
    (132, 68): (2.7815e-02, 3.2778e-03, 7.1459e-02, 7.1702e-02, 1.2724e-03),
}
# Table 6: SD N -> [(N1/N2, R_S)]
PAPER_RS = {127: [((63, 63), 3.27), ((63, 31), 4.5)], 255: [((127, 127), 6.46), ((127, 63), 9.26)],
            511: [((255, 255), 3.70), ((255, 127), 7.14)]}
IC = ((0.0, 0.0, 0.0), (1000.0, 100.0), (500.0, 50.0))


def dd_subdomains(N1, N2, dt):
    subs = []
    for sub, (N, r) in enumerate(((N1, R1), (N2, R2))):
        n, lo, hi, _ = paper_mesh(N, r)
        subs.append(api.CaseOneSubdomain(n, lo, hi, sub, R1, R2, 0, 0, dt))
    return subs


def sd_reference(Nref=516, steps=100, dt=1e-8):
    cfg = test_a_config(Nref, dt=dt, steps=steps)
    ctx = api.DPM.from_config(cfg)
    rho = torch.zeros((cfg.n,) * 3, dtype=torch.float64, device="cuda")
    c = torch.zeros_like(rho)
    ctx.pks_init(rho, c, cfg.ic_center, *cfg.ic_rho, *cfg.ic_c, rho_cell_average=True)
    logs = ctx.pks_step(rho, c, cfg.steps, chi=cfg.chi, dt_cap=dt, dt_rule=1, clamp=1)
    torch.cuda.synchronize()
    return rho, c, np.array([lg["rho_max_mplus"] for lg in logs]), ctx.info["h"]


def restrict_error(u, mp, n, r, h, uf, hf):
    """max over M+ of |u - mean of the fine values in the coarse cell| (R37)."""
    ratio = int(round(h / hf))
    assert abs(ratio * hf - h) < 1e-12 * h
    off = int(round((0.5 - r) / hf))                     # the fine mesh is the r = 0.5 box
    i, j, k = mp // (n * n), (mp // n) % n, mp % n
    base = [2 + off + (q - 2) * ratio for q in (i, j, k)]
    acc = torch.zeros(mp.shape, dtype=torch.float64, device="cuda")
    for a in range(ratio):
        for b in range(ratio):
            for d in range(ratio):
                acc += uf[base[0] + a, base[1] + b, base[2] + d]
    return float((u.reshape(-1)[mp] - acc / ratio ** 3).abs().max())


def run_tables(pairs=tuple(PAPER_DD), Nref=516, steps=100, dt=1e-8):
    rf, cf, Rser, hf = sd_reference(Nref, steps, dt)
    rows = []
    for N1, N2 in pairs:
        subs = dd_subdomains(N1, N2, dt)
        sol = DDSolver(subs, dt, dt_rule=1)
        sol.init(*IC, rho_cell_average=1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        logs = [sol.step() for _ in range(steps)]
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        S = np.array([lg["rho_max_mplus"] for lg in logs])
        e_rel = float(np.sqrt(np.sum((S - Rser) ** 2)) / np.sqrt(np.sum(Rser ** 2)))
        row = {"N1/N2": f"{N1}/{N2}", "h1/h2": f"1/{round(subs[1].info['h'] / subs[0].info['h'])}",
               "E_rel": e_rel, "wall_s": wall, "mass_drift": logs[-1]["mass"] / logs[0]["mass"] - 1.0}
        for name, (rho, c), o, r in zip(("Omega1", "Omega2"), sol.fields, subs, (R1, R2)):
            mp = torch.from_numpy(o.copy_set("mplus")).cuda()
            row[f"Einf_rho_{name}"] = restrict_error(rho, mp, o.n, r, o.info["h"], rf, hf)
            row[f"Einf_c_{name}"] = restrict_error(c, mp, o.n, r, o.info["h"], cf, hf)
        p = PAPER_DD.get((N1, N2))
        if p:
            row["paper"] = {"Einf_rho_Omega1": p[0], "Einf_rho_Omega2": p[1], "Einf_c_Omega1": p[2],
                            "Einf_c_Omega2": p[3], "E_rel": p[4]}
        rows.append(row)
        del sol, subs
    return {"test": "A-DD (Tables 1-3, DD columns)", "reference": f"SD N={Nref}, mean over the coarse cell",
            "rows": rows}


def _sd_wall(N, T, cap=1.0):
    """The SD run to T: the step count from a first pass, then the timed run as ONE dpm_pks_step call
    (the product's fastest SD path: speculative step graphs)."""
    cfg = test_a_config(N, dt=cap, steps=1)
    ctx = api.DPM.from_config(cfg)
    rho = torch.zeros((cfg.n,) * 3, dtype=torch.float64, device="cuda")
    c = torch.zeros_like(rho)
    ctx.pks_init(rho, c, cfg.ic_center, *cfg.ic_rho, *cfg.ic_c, rho_cell_average=True)
    t, steps = 0.0, 0
    while t < T:
        t = ctx.pks_step(rho, c, 1, chi=1.0, dt_cap=cap, dt_rule=0, clamp=1)[-1]["t"]
        steps += 1
    ctx.pks_init(rho, c, cfg.ic_center, *cfg.ic_rho, *cfg.ic_c, rho_cell_average=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    logs = ctx.pks_step(rho, c, steps, chi=1.0, dt_cap=cap, dt_rule=0, clamp=1)
    torch.cuda.synchronize()
    return time.perf_counter() - t0, steps, sum(lg["rebuilt"] for lg in logs)


def _dd_wall(N1, N2, T, cap=1.0):
    subs = dd_subdomains(N1, N2, cap)
    sol = DDSolver(subs, cap, dt_rule=0)
    sol.init(*IC, rho_cell_average=1)
    torch.cuda.synchronize()
    t0, steps = time.perf_counter(), 0
    while sol.t < T:
        sol.step()
        steps += 1
    torch.cuda.synchronize()
    return time.perf_counter() - t0, steps, sol.builds


def run_rs(T=6e-5, sizes=(127, 255)):
    rows = []
    for N in sizes:
        _sd_wall(N, T)                                   # warm-up (graph capture, plans)
        tsd, nsd, bsd = _sd_wall(N, T)
        for (N1, N2), paper in PAPER_RS[N]:
            _dd_wall(N1, N2, T)
            tdd, ndd, bdd = _dd_wall(N1, N2, T)
            rows.append({"SD N": N, "DD N1/N2": f"{N1}/{N2}", "T_SD_s": tsd, "T_DD_s": tdd, "R_S": tsd / tdd,
                         "paper_R_S (32-core CPU, P:939)": paper, "steps_SD": nsd, "steps_DD": ndd,
                         "builds_SD": bsd, "builds_DD": bdd})
    return {"test": "A (Table 6 R_S context)", "T": T, "rows": rows}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--tables", action="store_true")
    ap.add_argument("--rs", action="store_true")
    a = ap.parse_args()
    out = {}
    if a.tables or not a.rs:
        out["tables"] = run_tables()
    if a.rs:
        out["rs"] = run_rs()
    print(json.dumps(out))
