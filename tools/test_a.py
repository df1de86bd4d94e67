"""The paper's Test A convergence of the max density (P:662-666 eq. sd-conv-max-density-in-space,
Table 3 at P:786-805), single domain, on one GPU.

For each mesh N (paper convention) runs 100 PKS steps at the fixed dt = 1e-8 to T = 1e-6
and records ||ρ^i||∞ over M+  per step.  The reference series is the paper's, the N = 516
run, when 516 is the finest mesh requested (the default); otherwise the Richardson extrapolation
(second order, h halves between the paper's meshes) of the two finest meshes run; and

    E_rel(N) = sqrt(Σ_i (||ρ^i_N||∞ - R_i)^2 Δt) / sqrt(Σ_i R_i^2 Δt)

is compared with the paper's E_rel (SD column of Table 3): 1.0196e-01 (36), 2.6378e-02 (68),
6.3461e-03 (132), 1.2724e-03 (260).

    python tools/test_a.py [--N 36 68 132 260 516]
    python tools/test_a.py --time [--N 255]        # Tables 4-5: convergence in time

Convergence in time (P:667-670 eq. sd-conv-in-time, Tables 4-5 at P:812-870): on the fixed mesh
N = 255, dt = 1e-7/τ (τ = 16 ... 256) to T = 1e-6, E_t = max over M+ of |ρ_τ - ρ_ref| (and c) at
T against the run at τ* = 512 (the printed rates 1.05 / 1.10 / 1.22 / 1.58 are exactly
log2((1/τ - 1/512)/(1/2τ - 1/512)), so the paper's reference is dt* = 1e-7/512).
Paper (SD): E_t(ρ) 8.2335e-03 / 3.9846e-03 / 1.8596e-03 / 7.9700e-04 / 2.6567e-04,
            E_t(c) 6.1248e-08 / 2.9665e-08 / 1.3889e-08 / 5.9737e-09 / 2.0236e-09.
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

from dpm_inputs import test_a_config  # noqa: E402
from paper_1811_03557_b200 import api  # noqa: E402

PAPER_E_REL = {36: 1.0196e-01, 68: 2.6378e-02, 132: 6.3461e-03, 260: 1.2724e-03}
PAPER_E_T_RHO = {16: 8.2335e-03, 32: 3.9846e-03, 64: 1.8596e-03, 128: 7.9700e-04, 256: 2.6567e-04}
PAPER_E_T_C = {16: 6.1248e-08, 32: 2.9665e-08, 64: 1.3889e-08, 128: 5.9737e-09, 256: 2.0236e-09}


IC_CELL = True   # ρ̄0 as cell averages (R36, the paper's reading: Table 3 to ~0.1%); False: node values (R14)


def series(N):
    cfg = test_a_config(N)
    ctx = api.DPM.from_config(cfg)
    rho = torch.zeros((cfg.n,) * 3, dtype=torch.float64, device="cuda")
    c = torch.zeros_like(rho)
    ctx.pks_init(rho, c, cfg.ic_center, *cfg.ic_rho, *cfg.ic_c, rho_cell_average=IC_CELL)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    logs = ctx.pks_step(rho, c, cfg.steps, chi=cfg.chi, dt_cap=cfg.dt, dt_rule=1, clamp=1)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    s = np.array([lg["rho_max_mplus"] for lg in logs])
    return s, {"N": N, "h": ctx.info["h"], "K": ctx.K, "rho_max_T": float(s[-1]), "t_end": logs[-1]["t"],
               "mass_drift": logs[-1]["mass"] / logs[0]["mass"] - 1.0, "wall_s": wall}


def run(Ns=(36, 68, 132, 260, 516)):
    Ns = sorted(Ns)
    S, info = {}, {}
    for N in Ns:
        S[N], info[N] = series(N)
    f, c = Ns[-1], Ns[-2]
    if f == 516:                            # the paper's reference mesh (Tables 1-3)
        R, ref = S[f], "N=516 (the paper's reference)"
        Ns = Ns[:-1]
    else:
        R = (4.0 * S[f] - S[c]) / 3.0      # Richardson, p = 2, h_c = 2 h_f
        ref = f"Richardson of N={c} and N={f} (the paper's: N=516)"
    rows = []
    for N in Ns:
        e = float(np.sqrt(np.sum((S[N] - R) ** 2)) / np.sqrt(np.sum(R ** 2)))
        rows.append(dict(info[N], E_rel=e, paper_E_rel=PAPER_E_REL.get(N)))
    for a, b in zip(rows, rows[1:]):
        b["rate"] = math.log2(a["E_rel"] / b["E_rel"]) if b["E_rel"] > 0 else None
    return {"test": "A", "reference": ref, "ic": "cell averages (R36)" if IC_CELL else "node values (R14)",
            "rows": rows, "reference_run": info[f] if f == 516 else None}


PAPER_EINF_RHO = {36: 1.4046e+00, 68: 3.6990e-01, 132: 1.2224e-01, 260: 2.7815e-02}
PAPER_EINF_C = {36: 5.6759e+00, 68: 1.4766e+00, 132: 3.5615e-01, 260: 7.1459e-02}


def run_einf(Ns=(36, 68, 132, 260), Nref=516, restrict="cell"):
    """Tables 1-2 (P:650-655 eq. sd-error-in-max-norm): E∞ = max over the coarse M+ of |ρ̄_h - ρ̄_h*| at
    T = 1e-6 (and for c).  The paper's meshes do not nest, but every coarse node sits at the centre of a
    2x2x2 cell of the N = 516 mesh (fine index ratio (i - 3/2) + 3/2 is a half-integer for the even
    ratios 16/8/4/2), so the reference is read there by trilinear interpolation = the 8-point mean."""
    def state(N):
        cfg = test_a_config(N)
        ctx = api.DPM.from_config(cfg)
        rho = torch.zeros((cfg.n,) * 3, dtype=torch.float64, device="cuda")
        c = torch.zeros_like(rho)
        ctx.pks_init(rho, c, cfg.ic_center, *cfg.ic_rho, *cfg.ic_c, rho_cell_average=IC_CELL)
        ctx.pks_step(rho, c, cfg.steps, chi=cfg.chi, dt_cap=cfg.dt, dt_rule=1, clamp=1)
        torch.cuda.synchronize()
        return rho, c, torch.from_numpy(ctx.copy_set("mplus")).cuda()

    rf, cf, _ = state(Nref)
    rows = []
    for N in Ns:
        rc, cc, mp = state(N)
        ratio = (Nref - 4) // (N - 4)
        assert ratio * (N - 4) == Nref - 4 and ratio % 2 == 0
        i, j, k = mp // (N * N), (mp // N) % N, mp % N
        if restrict == "cell":   # mean of the ratio^3 fine values inside the coarse cell
            w = ratio
            base = [ratio * q - 2 * ratio + 2 for q in (i, j, k)]
        else:                    # trilinear at the coarse node = mean of the surrounding 2x2x2
            w = 2
            base = [ratio * q - (3 * ratio) // 2 + 1 for q in (i, j, k)]
        out = {"N": N}
        for name, fc, ff, paper in (("rho", rc, rf, PAPER_EINF_RHO), ("c", cc, cf, PAPER_EINF_C)):
            acc = torch.zeros(mp.shape, dtype=torch.float64, device="cuda")
            for a in range(w):
                for b in range(w):
                    for d in range(w):
                        acc += ff[base[0] + a, base[1] + b, base[2] + d]
            e = float((fc.reshape(-1)[mp] - acc / w ** 3).abs().max())
            out[f"Einf_{name}"], out[f"paper_Einf_{name}"] = e, paper.get(N)
        rows.append(out)
    for a, b in zip(rows, rows[1:]):
        for name in ("rho", "c"):
            b[f"rate_{name}"] = math.log2(a[f"Einf_{name}"] / b[f"Einf_{name}"])
    how = "mean over the coarse cell" if restrict == "cell" else "8-point (trilinear) mean at the coarse nodes"
    return {"test": "A-Einf", "reference": f"N={Nref}, {how}", "rows": rows}


def final_state(N, tau, T=1e-6, dT=1e-7, coupling=0):
    dt = dT / tau
    cfg = test_a_config(N, dt=dt, steps=int(round(T / dt)))
    ctx = api.DPM.from_config(cfg)
    rho = torch.zeros((cfg.n,) * 3, dtype=torch.float64, device="cuda")
    c = torch.zeros_like(rho)
    ctx.pks_init(rho, c, cfg.ic_center, *cfg.ic_rho, *cfg.ic_c, rho_cell_average=IC_CELL)
    t0 = time.perf_counter()
    logs = ctx.pks_step(rho, c, cfg.steps, chi=cfg.chi, dt_cap=dt, dt_rule=1, clamp=1, coupling=coupling)
    torch.cuda.synchronize()
    mp = torch.from_numpy(ctx.copy_set("mplus")).cuda()
    return rho.reshape(-1)[mp], c.reshape(-1)[mp], logs[-1]["t"], time.perf_counter() - t0


def run_time(N=255, taus=(16, 32, 64, 128, 256), tau_ref=512, T=1e-6, dT=1e-7, coupling=0):
    rr, cr, tr, wr = final_state(N, tau_ref, T, dT, coupling)
    rows = []
    for tau in taus:
        r, c, t, w = final_state(N, tau, T, dT, coupling)
        rows.append({"tau": tau, "dt": dT / tau, "t_end": t, "wall_s": w,
                     "E_t_rho": float((r - rr).abs().max()), "paper_E_t_rho": PAPER_E_T_RHO.get(tau),
                     "E_t_c": float((c - cr).abs().max()), "paper_E_t_c": PAPER_E_T_C.get(tau)})
    for a, b in zip(rows, rows[1:]):
        b["rate_rho"] = math.log2(a["E_t_rho"] / b["E_t_rho"])
        b["rate_c"] = math.log2(a["E_t_c"] / b["E_t_c"])
    return {"test": "A-time", "N": N, "tau_ref": tau_ref, "t_end_ref": tr, "wall_ref_s": wr, "rows": rows}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, nargs="+", default=None)
    ap.add_argument("--time", action="store_true")
    ap.add_argument("--einf", action="store_true", help="Tables 1-2: nodewise E∞ against N = 516")
    ap.add_argument("--ic", choices=["cell", "point"], default="cell",
                    help="ρ̄0 on M+ \\ γ: cell averages (R36, default) or node values (R14)")
    a = ap.parse_args()
    IC_CELL = a.ic == "cell"
    if a.einf:
        print(json.dumps(run_einf()))
    elif a.time:
        print(json.dumps(run_time(a.N[0] if a.N else 255)))
    else:
        print(json.dumps(run(a.N or [36, 68, 132, 260, 516])))
