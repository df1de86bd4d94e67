"""PKS time stepping — oracle (test infrastructure only).

Transcribes, cell by cell, the hybrid finite-volume / finite-difference IMEX scheme
 and the algorithm outline Steps 1-8, with the readings of
SURVEY.md §8(c) R13-R20 (listed in DESIGN.md):

* face gradient of c: (c_{j+1} - c_j)/h (`eqn:c-central-difference`);
* minmod (`eqn:slope_limiter`) of (2Δ+/h, Δ0/(2h), 2Δ-/h);
  R15: the slope of a cell is 0 along an axis unless both neighbours are in N+;
* upwind face value: left reconstruction if ∇c > 0, else the right one (R16);
* g = Σ_axes (χ ρ_{+½} ∇c_{+½} - χ ρ_{-½} ∇c_{-½})/h;
* f_ρ = ρ̄ - dt g,  f_c = (1 - dt) c + dt ρ̄ on M+ (P:89-96);
* CFL (`eqn:cfl_condition`) over faces with an endpoint in M+ (R19);
* dt_i = min(dt_{i-1}, dt_cap, CFL, 0.5 h^2) (Step 3 P:427 + R13), BEP rebuilt iff
  dt strictly decreases (Step 4b P:431);
* Steps 4a-7: particular solves, reduced BEP by least squares, u_γ = E C clamped at 0
  (R17), one combined Green's-formula solve restricted to N+ (R20);
* mass = h^3 Σ_{M+} ρ̄ (R18).
State: ρ̄ and c as [n][n][n] arrays holding values on N+ ∩ M0 (0 elsewhere); ghost
nodes of N+ hold 0 (Dirichlet AP, R5).
"""
import math

import numpy as np
import scipy.special

from . import ap, dpm, grid


def minmod(*xs):
    """minmod(x_1..x_M): min if all > 0, max if all < 0, else 0 (elementwise)."""
    X = np.stack(np.broadcast_arrays(*[np.asarray(x, dtype=np.float64) for x in xs]))
    return np.where((X > 0).all(axis=0), X.min(axis=0), np.where((X < 0).all(axis=0), X.max(axis=0), 0.0))


def _pad(u):
    n = u.shape[-1]
    p = np.zeros((n + 2,) * 3)
    p[1:-1, 1:-1, 1:-1] = u
    return p


def _shift(p, ax, s):
    """Value at lattice index + s along axis ax (out-of-lattice -> 0 / False)."""
    out = np.zeros_like(p)
    src = [slice(None)] * 3
    dst = [slice(None)] * 3
    if s == 1:
        src[ax] = slice(1, None)
        dst[ax] = slice(0, -1)
    else:
        src[ax] = slice(0, -1)
        dst[ax] = slice(1, None)
    out[tuple(dst)] = p[tuple(src)]
    return out


def limited_slopes(rho_lat: np.ndarray, nplus_lat: np.ndarray, h: float):
    """Per-axis minmod slopes on the (n+2)^3 lattice (R15)."""
    sl = []
    for ax in range(3):
        rp, rm = _shift(rho_lat, ax, 1), _shift(rho_lat, ax, -1)
        okp, okm = _shift(nplus_lat, ax, 1), _shift(nplus_lat, ax, -1)
        s = minmod(2.0 * (rp - rho_lat) / h, (rp - rm) / (2.0 * h), 2.0 * (rho_lat - rm) / h)
        sl.append(np.where(okp & okm & nplus_lat, s, 0.0))
    return sl


def convection(rho: np.ndarray, c: np.ndarray, ps: grid.PointSets, h: float, chi: float) -> np.ndarray:
    """g on M+ (P:98-119), as an [n][n][n] array (0 off M+)."""
    R = _pad(rho)
    Cl = _pad(c)
    npl = ps.nplus_lat
    S = limited_slopes(R, npl, h)
    g = np.zeros_like(R)
    for ax in range(3):
        Rp, Rm = _shift(R, ax, 1), _shift(R, ax, -1)
        Sp, Sm = _shift(S[ax], ax, 1), _shift(S[ax], ax, -1)
        Cp, Cm = _shift(Cl, ax, 1), _shift(Cl, ax, -1)
        gE = (Cp - Cl) / h
        gW = (Cl - Cm) / h
        rhoE = np.where(gE > 0, R + 0.5 * h * S[ax], Rp - 0.5 * h * Sp)
        rhoW = np.where(gW > 0, Rm + 0.5 * h * Sm, R - 0.5 * h * S[ax])
        g += (chi * rhoE * gE - chi * rhoW * gW) / h
    g = g[1:-1, 1:-1, 1:-1]
    return np.where(ps.mplus, g, 0.0)


def assemble_rhs(rho, c, g, dt):
    """f_ρ = ρ̄ - dt g, f_c = (1 - dt) c + dt ρ̄."""
    return rho - dt * g, (1.0 - dt) * c + dt * rho


def cfl_dt(c: np.ndarray, ps: grid.PointSets, h: float, chi: float) -> float:
    """min over axes of h/(6 χ max|∇c|) over faces of M+ cells (R19); inf if flat."""
    Cl = _pad(c)
    mp = np.zeros_like(ps.nplus_lat)
    mp[1:-1, 1:-1, 1:-1] = ps.mplus
    best = np.inf
    for ax in range(3):
        gE = np.abs(_shift(Cl, ax, 1) - Cl) / h
        gW = np.abs(Cl - _shift(Cl, ax, -1)) / h
        mx = max(gE[mp].max(initial=0.0), gW[mp].max(initial=0.0))
        if mx > 0:
            best = min(best, h / (6.0 * chi * mx))
    return best


class PKSOracle:
    """Steps 1-8 for one single-domain configuration."""

    def __init__(self, cfg, dt_rule: int = 0, clamp: bool = True, coupling: int = 0):
        self.cfg = cfg
        self.g, self.ps = grid.point_sets_for(cfg)
        self.E, self.d, self.unit, self.foot = dpm.extension_matrix(
            self.g, self.ps, cfg.kind, cfg.center, cfg.semi, cfg.lmax, cfg.basis)
        self.gin_pos = np.searchsorted(self.ps.list("gamma"), self.ps.list("gamma_in"))
        self.dt_rule = dt_rule
        self.clamp = clamp
        self.coupling = coupling   # 1: the c equation uses ρ̄^{i+1} (sequential; not the printed P:89-96)
        self.dt_prev = np.inf
        self.dt_bep = None
        self.B = None
        self.builds = 0
        self.t = 0.0

    def initial_state(self, rho_cell_average: bool = False):
        """R14: IC at the node on M+ \\ γ, at the foot point on γ; 0 elsewhere.  With rho_cell_average
        (R36; the paper evolves cell averages ρ̄), ρ̄ on M+ \\ γ is the average of ρ0 over the cell
        [x - h/2, x + h/2]^3: for A exp(-a |x - x0|^2) the product over the axes of
        sqrt(π/a) (erf(√a (s + h/2)) - erf(√a (s - h/2))) / (2h), s = x - x0."""
        cfg, g, ps = self.cfg, self.g, self.ps
        n = g.n
        x = g.coords()
        X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
        c0 = np.asarray(cfg.ic_center)

        def ic(A, a, XX, YY, ZZ):
            return A * np.exp(-a * ((XX - c0[0]) ** 2 + (YY - c0[1]) ** 2 + (ZZ - c0[2]) ** 2))

        rho = np.where(ps.nplus, ic(*cfg.ic_rho, X, Y, Z), 0.0)
        if rho_cell_average:
            A, a = cfg.ic_rho
            h = g.h

            def avg1(s):
                if a <= 0:
                    return np.ones_like(s)
                q = math.sqrt(a)
                return math.sqrt(math.pi / a) * (scipy.special.erf(q * (s + h / 2)) - scipy.special.erf(q * (s - h / 2))) / (2 * h)

            cell = A * avg1(X - c0[0]) * avg1(Y - c0[1]) * avg1(Z - c0[2])
            rho = np.where(ps.mplus, cell, rho)    # γ_in values are overwritten by the foot values below
        c = np.where(ps.nplus, ic(*cfg.ic_c, X, Y, Z), 0.0)
        gidx = ps.list("gamma")
        F = self.foot
        rho.reshape(-1)[gidx] = ic(*cfg.ic_rho, F[:, 0], F[:, 1], F[:, 2])
        c.reshape(-1)[gidx] = ic(*cfg.ic_c, F[:, 0], F[:, 1], F[:, 2])
        return rho, c

    def build(self, dt):
        _, self.B, _ = dpm.projection_and_bep(self.E, self.g, self.ps, dt)
        self.dt_bep = dt
        self.builds += 1

    def step(self, rho, c):
        cfg, g, ps, h = self.cfg, self.g, self.ps, self.g.h
        if self.dt_rule == 0:
            dt = min(self.dt_prev, cfg.dt, cfl_dt(c, ps, h, cfg.chi), 0.5 * h * h)   # Step 3 + R13
        else:
            dt = cfg.dt
        rebuilt = False
        if self.B is None or dt != self.dt_bep:                                     # Step 2 / 4b
            self.build(dt)
            rebuilt = True
        gconv = convection(rho, c, ps, h, cfg.chi)
        f_rho, f_c = assemble_rhs(rho, c, gconv, dt)                                # Step 4a
        out = []
        us = []
        resid, clamp_max = 0.0, 0.0
        for r in range(2):
            if r == 1 and self.coupling == 1:
                _, f_c = assemble_rhs(out[0], c, gconv, dt)                         # c from ρ̄^{i+1}
            f = (f_rho, f_c)[r]
            up = ap.solve(dpm.particular_rhs(f, ps, dt), h, dt)                      # G f
            rhs = up.reshape(-1)[ps.list("gamma_in")]
            C = dpm.lstsq(self.B, rhs)                                              # Step 5
            resid = max(resid, np.linalg.norm(self.B @ C - rhs) / np.linalg.norm(rhs))   # BEP LSQ residual
            u_gamma = self.E @ C
            clamp_max = max(clamp_max, float(np.max(np.maximum(-u_gamma, 0.0))))     # R17 clamp magnitude
            if self.clamp:
                u_gamma = np.maximum(u_gamma, 0.0)                                  # R17
            out.append(dpm.green(u_gamma, f, g, ps, dt))                            # Steps 6-7 (R20)
            us.append(u_gamma)
        self.dt_prev = dt
        self.t += dt
        return out[0], out[1], dict(dt=dt, rebuilt=rebuilt, t=self.t, lsq_resid=resid, clamp_max=clamp_max)

    def mass(self, rho):
        h = self.g.h
        return h ** 3 * rho[self.ps.mplus].sum()                                    # R18

    def run(self, nsteps=None):
        rho, c = self.initial_state()
        logs = []
        for _ in range(nsteps if nsteps is not None else self.cfg.steps):
            rho, c, log = self.step(rho, c)
            log["mass"] = self.mass(rho)
            logs.append(log)
        return rho, c, logs


def diagnostics(rho: np.ndarray, c: np.ndarray, g: grid.Grid, ps: grid.PointSets, center) -> dict:
    """Mass (R18), second moment M_h (eq. sd-norm:second-moment) and free energy E_h
    (eq. sd-norm:free-energy) of a state on M+, literally:
      M_h = Σ_{M+} h^3 |x - x_c|^2 ρ̄,
      E_h = Σ_{M+} h^3 { ρ̄ ln ρ̄ - ρ̄ c + c^2/2 + [(c_{j+1}-c_{j-1})^2 + (c_{k+1}-c_{k-1})^2
                                                  + (c_{l+1}-c_{l-1})^2] / (8 h^2) }.
    Readings (R35): |x - x_c| from the domain centre (the paper's domain is centred at the origin);
    ρ̄ ln ρ̄ := 0 for ρ̄ <= 0 (its limit at 0); c at ghost nodes is 0 (the state's ghost values)."""
    h = g.h
    x = g.coords()
    X, Y, Z = np.meshgrid(x - center[0], x - center[1], x - center[2], indexing="ij")
    m = ps.mplus
    r, cc = rho[m], c[m]
    second = h ** 3 * np.sum((X[m] ** 2 + Y[m] ** 2 + Z[m] ** 2) * r)
    cp = np.zeros(tuple(s + 2 for s in c.shape))
    cp[1:-1, 1:-1, 1:-1] = c
    gx = cp[2:, 1:-1, 1:-1] - cp[:-2, 1:-1, 1:-1]
    gy = cp[1:-1, 2:, 1:-1] - cp[1:-1, :-2, 1:-1]
    gz = cp[1:-1, 1:-1, 2:] - cp[1:-1, 1:-1, :-2]
    rlnr = np.where(r > 0, r * np.log(np.where(r > 0, r, 1.0)), 0.0)
    grad = (gx[m] ** 2 + gy[m] ** 2 + gz[m] ** 2) / (8.0 * h * h)
    free = h ** 3 * np.sum(rlnr - r * cc + 0.5 * cc * cc + grad)
    return {"mass": h ** 3 * np.sum(r), "second_moment": second, "free_energy": free}
