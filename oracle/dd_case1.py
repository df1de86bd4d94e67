"""The paper's two-subdomain DPM domain decomposition, Case 1 (Z ∩ Γ = ∅) — oracle (test
infrastructure only).

Section "A Domain Decomposition approach based on DPM" with the numerical setup of
P:594-641, literally:
* Ω = ball of radius r2 (= 0.5) centred at the origin; Ω1 = ball of radius r1 (= 0.25) and
  Ω2 = the shell r1 < |x| < r2; the artificial interface Z = {|x| = r1}.
* Each Ω_ℓ is embedded in its own auxiliary cube [-r_ℓ - 2h_ℓ, r_ℓ + 2h_ℓ]^3 with N_ℓ cells,
  h_ℓ = 2 r_ℓ / (N_ℓ - 4) ("N1/N2" P:627), i.e. dpm_inputs.paper_mesh(N_ℓ, r_ℓ).
* Point sets of Definition 1 per subdomain (exact rationals, R6); the discrete grid
  interface ζ1 = γ of Ω1; the discrete boundary of Ω2, N2+ ∩ N2-, splits into ζ2 (near Z) and
  γ (near Γ) (reading R38: a point belongs to the nearer of the two spheres).
* Extension operators with the paper's zonal basis φ_ν = P_ν(cos θ):
  on Γ the zero-Neumann 3-term operator {φ_ν, (d²/2) φ_ν}, d = |x| - r2; on Z the
  full 3-term operator with the interface Cauchy data {φ_ν, d φ_ν, (d²/2) φ_ν}, d = |x| - r1 along
  the one normal of Z (+r̂), whose coefficients are SHARED by Ω1 and Ω2 — the interface conditions
  ∂^k u1/∂n^k = ∂^k u2/∂n^k, k = 0, 1, 2 (`eqn:interface_condition` P:477-480).
  Global unknowns C = [Z: C⁰ | C¹ | C² (Mz+1 each) | Γ: C⁰ | C² (Mg+1 each)], K = 3(Mz+1) + 2(Mg+1).
* Coupled reduced BEPs (`eqn:reduced_DD1_BEP1` P:527, `eqn:reduced_DD1_BEP2` P:535-547): rows on
  ζ1,in for Ω1 and on γ_in ∪ ζ2,in for Ω2, each row E[p] - Tr_p P (E on the subdomain's discrete
  boundary); the two row blocks are stacked into one least-squares problem (columns equilibrated
  to unit 2-norm, as R24), solved by numpy.linalg.lstsq.
* PKS step (Steps 3-7 P:427-437) in each subdomain with its own grid, one global Δt
  (R13 with the minimum over both subdomains of the CFL bound and 0.5 h_ℓ²), u = max(E C, 0) on
  each discrete boundary (R17) and the Green's formula per subdomain (R20).
* Initial data (R38): as R14 on γ (the IC at the foot on Γ); at ζ points (interior points of Ω on
  either side of Z) the IC at the node — or, for ρ̄ with cell averages (R36), the cell average, as
  on the rest of M_ℓ+.
"""
from dataclasses import dataclass
from typing import List

import math

import numpy as np
import scipy.special

from . import ap, dpm, grid, pks, sh

Z_PIECE, G_PIECE = 0, 1


@dataclass
class Subdomain:
    name: str                 # "ball" (Ω1) or "shell" (Ω2)
    g: grid.Grid
    ps: grid.PointSets
    piece: np.ndarray         # per γ-list point: Z_PIECE or G_PIECE
    E: np.ndarray             # |γ| x K extension rows (each point's own piece block, 0 elsewhere)
    foot: np.ndarray          # |γ| x 3 foot on the point's own sphere
    d: np.ndarray             # |γ| signed distance to the point's own sphere (+ along +r̂)
    gin_pos: np.ndarray       # positions of γ_in inside the γ list (the BEP rows)


def column_blocks(Mz: int, Mg: int):
    """Z block [0, 3(Mz+1)), Γ block [3(Mz+1), K)."""
    kz = 3 * (Mz + 1)
    return slice(0, kz), slice(kz, kz + 2 * (Mg + 1)), kz + 2 * (Mg + 1)


def extension_rows(P: np.ndarray, piece: np.ndarray, r1: float, r2: float, Mz: int, Mg: int):
    """E (|P| x K), foot, d for points P whose sphere is given by `piece`."""
    zb, gb, K = column_blocks(Mz, Mg)
    rad = np.sqrt((P ** 2).sum(axis=1))
    unit = P / rad[:, None]
    E = np.zeros((len(P), K))
    foot = np.empty_like(P)
    d = np.empty(len(P))
    isz = piece == Z_PIECE
    for r, m, M, blk in ((r1, isz, Mz, zb), (r2, ~isz, Mg, gb)):
        if not m.any():
            continue
        dd = rad[m] - r
        phi = sh.zonal(M, unit[m])
        if blk is zb:       # full 3-term interface operator: u, ∂_n u, ∂²_n u unknown
            cols = np.concatenate([phi, dd[:, None] * phi, 0.5 * (dd ** 2)[:, None] * phi], axis=1)
        else:               # zero Neumann on Γ: the d term vanishes
            cols = np.concatenate([phi, 0.5 * (dd ** 2)[:, None] * phi], axis=1)
        E[np.ix_(np.flatnonzero(m), np.arange(blk.start, blk.stop))] = cols
        foot[m] = r * unit[m]
        d[m] = dd
    return E, foot, d


def make_subdomain(name: str, N: int, r1: float, r2: float, Mz: int, Mg: int) -> Subdomain:
    from dpm_inputs import paper_mesh
    n, lo, hi, _ = paper_mesh(N, r1 if name == "ball" else r2)
    g = grid.Grid(n, lo, hi)
    if name == "ball":
        mask = grid.inside_mask(g, "sphere", (0.0, 0.0, 0.0), (r1, r1, r1))
    else:
        mask = grid.shell_inside_mask(g, r1, r2)
    ps = grid.point_sets_from_mask(g, mask)
    P = dpm.gamma_points(g, ps)
    rad = np.sqrt((P ** 2).sum(axis=1))
    if name == "ball":
        piece = np.full(len(P), Z_PIECE)
    else:   # R38: the nearer sphere (the two layers are (r2 - r1)/h2 - O(1) nodes apart)
        piece = np.where(np.abs(rad - r1) < np.abs(rad - r2), Z_PIECE, G_PIECE)
    E, foot, d = extension_rows(P, piece, r1, r2, Mz, Mg)
    gin_pos = np.searchsorted(ps.list("gamma"), ps.list("gamma_in"))
    return Subdomain(name, g, ps, piece, E, foot, d, gin_pos)


def bep_rows(sub: Subdomain, dt: float) -> np.ndarray:
    """Reduced BEP rows of one subdomain: E[γ_in] - Tr_γin P_{N+γ} E  (P:527-547 with P:283-290)."""
    PgE = dpm.potential_trace(sub.E, sub.g, sub.ps, dt, sub.ps.list("gamma"))
    return sub.E[sub.gin_pos] - PgE[sub.gin_pos]


def stacked_lstsq(Bs: List[np.ndarray], gs: List[np.ndarray]) -> np.ndarray:
    """C = argmin || [B1; B2] C - [g1; g2] ||, columns equilibrated to unit 2-norm (as R24)."""
    Bst = np.concatenate(Bs, axis=0)
    gst = np.concatenate(gs, axis=0)
    D = 1.0 / np.linalg.norm(Bst, axis=0)
    y = np.linalg.lstsq(Bst * D, gst, rcond=None)[0]
    return D[:, None] * y if y.ndim > 1 else D * y


class CaseOneDD:
    """Two-subdomain PKS (Steps 1-8) on Ω1 (ball r1, N1 cells) and Ω2 (shell, N2 cells)."""

    def __init__(self, N1: int, N2: int, dt_cap: float, steps: int, r1: float = 0.25, r2: float = 0.5,
                 Mz: int = 0, Mg: int = 0, chi: float = 1.0, dt_rule: int = 0, clamp: bool = True,
                 rho_ic=(1000.0, 100.0), c_ic=(500.0, 50.0), rho_cell_average: bool = False):
        self.subs = [make_subdomain("ball", N1, r1, r2, Mz, Mg), make_subdomain("shell", N2, r1, r2, Mz, Mg)]
        self.r1, self.r2, self.Mz, self.Mg = r1, r2, Mz, Mg
        self.K = column_blocks(Mz, Mg)[2]
        self.dt_cap, self.steps, self.chi, self.dt_rule, self.clamp = dt_cap, steps, chi, dt_rule, clamp
        self.rho_ic, self.c_ic, self.rho_cell_average = rho_ic, c_ic, rho_cell_average
        self.dt_prev, self.dt_bep, self.Bs, self.builds, self.t = np.inf, None, None, 0, 0.0

    def initial_state(self):
        """R38 (module docstring): Gaussians centred at the origin (Test A)."""
        out = []
        for s in self.subs:
            n, h = s.g.n, s.g.h
            x = s.g.coords()
            X, Y, Z = np.meshgrid(x, x, x, indexing="ij")

            def gauss(A, a, XX, YY, ZZ):
                return A * np.exp(-a * (XX ** 2 + YY ** 2 + ZZ ** 2))

            rho = np.where(s.ps.nplus, gauss(*self.rho_ic, X, Y, Z), 0.0)
            c = np.where(s.ps.nplus, gauss(*self.c_ic, X, Y, Z), 0.0)
            if self.rho_cell_average:   # R36 on M+ and on the interface points
                A, a = self.rho_ic
                q = math.sqrt(a)

                def avg1(t):
                    return math.sqrt(math.pi / a) * (scipy.special.erf(q * (t + h / 2))
                                                     - scipy.special.erf(q * (t - h / 2))) / (2 * h)

                cell = A * avg1(X) * avg1(Y) * avg1(Z)
                zeta = np.zeros(n ** 3, dtype=bool)
                zeta[s.ps.list("gamma")[s.piece == Z_PIECE]] = True
                rho = np.where(s.ps.mplus | zeta.reshape(n, n, n), cell, rho)
            gidx = s.ps.list("gamma")[s.piece == G_PIECE]          # γ near Γ: IC at the foot (R14)
            F = s.foot[s.piece == G_PIECE]
            rho.reshape(-1)[gidx] = gauss(*self.rho_ic, F[:, 0], F[:, 1], F[:, 2])
            c.reshape(-1)[gidx] = gauss(*self.c_ic, F[:, 0], F[:, 1], F[:, 2])
            out.append((rho, c))
        return out

    def build(self, dt: float):
        self.Bs = [bep_rows(s, dt) for s in self.subs]
        self.dt_bep = dt
        self.builds += 1

    def step(self, state):
        chi = self.chi
        if self.dt_rule == 0:
            dt = min(self.dt_prev, self.dt_cap)
            for s, (_, c) in zip(self.subs, state):                 # Step 3 + R13, global minimum
                dt = min(dt, pks.cfl_dt(c, s.ps, s.g.h, chi), 0.5 * s.g.h ** 2)
        else:
            dt = self.dt_cap
        rebuilt = False
        if self.Bs is None or dt != self.dt_bep:                       # Step 2 / 4b
            self.build(dt)
            rebuilt = True
        frhs = []
        for s, (rho, c) in zip(self.subs, state):
            gconv = pks.convection(rho, c, s.ps, s.g.h, chi)
            frhs.append(pks.assemble_rhs(rho, c, gconv, dt))        # Step 4a
        new = [[None, None] for _ in self.subs]
        for fi in range(2):
            gs = []
            for s, fr in zip(self.subs, frhs):
                up = ap.solve(dpm.particular_rhs(fr[fi], s.ps, dt), s.g.h, dt)
                gs.append(up.reshape(-1)[s.ps.list("gamma_in")])
            C = stacked_lstsq(self.Bs, gs)                              # Step 5, coupled BEPs
            for k, (s, fr) in enumerate(zip(self.subs, frhs)):
                ug = s.E @ C
                if self.clamp:
                    ug = np.maximum(ug, 0.0)                            # R17
                new[k][fi] = dpm.green(ug, fr[fi], s.g, s.ps, dt)       # Steps 6-7 (R20)
        self.dt_prev = dt
        self.t += dt
        return [tuple(x) for x in new], dict(dt=dt, rebuilt=rebuilt, t=self.t, C=C)

    def mass(self, state):
        return sum(s.g.h ** 3 * rho[s.ps.mplus].sum() for s, (rho, _) in zip(self.subs, state))

    def run(self, nsteps=None):
        state = self.initial_state()
        logs = []
        for _ in range(nsteps if nsteps is not None else self.steps):
            state, log = self.step(state)
            log["mass"] = self.mass(state)
            logs.append(log)
        return state, logs


def coupled_elliptic_solve(dd: CaseOneDD, f_boxes, dt: float):
    """One coupled solve of (I - dt Δ) u = f on Ω1 ∪ Ω2 (zero Neumann on Γ, continuity of u, ∂_n u and
    ∂²_n u across Z), f given on each subdomain's box: the elliptic core of the step (pins)."""
    Bs = [bep_rows(s, dt) for s in dd.subs]
    gs = []
    for s, f in zip(dd.subs, f_boxes):
        up = ap.solve(dpm.particular_rhs(f, s.ps, dt), s.g.h, dt)
        gs.append(up.reshape(-1)[s.ps.list("gamma_in")])
    C = stacked_lstsq(Bs, gs)
    return [dpm.green(s.E @ C, f, s.g, s.ps, dt) for s, f in zip(dd.subs, f_boxes)], C
