"""Octant domain decomposition (config 5) — oracle (test infrastructure only).

The paper's DPM domain decomposition couples subdomains through boundary equations
that share the interface Cauchy data (interface condition `eqn:interface_condition` P:477-480);
at points near several boundary pieces it duplicates the equations and uses an averaged
"effective" density (Case 2).  Config 5's eight-octant split is not in the paper;
this module follows SURVEY.md §8(c) R24, R25, R31 literally:

* subdomain s = sign octant σ ∩ unit ball, in its canonical frame p (x_phys = σ ⊙ p) on the box
  [-0.1, 1.1]^3 (R3), point sets by Definition 1 on the exact octant mask;
* boundary pieces: the cap (octant of Γ, zero Neumann: {Y_ν, (d^2/2) Y_ν}, ν < (Lc+1)^2, ONE global
  expansion shared by all octants) and the three coordinate-plane quarter discs (each ONE global
  basis φ_jk(s, t) = P_j(s) P_k(t), j + k <= Li, over the unit disc, 2-term Cauchy data
  {φ, d φ} with d measured along +e_a, R25).  Columns:
  [cap Y | cap d^2/2 Y | plane x: φ, dφ | plane y: φ, dφ | plane z: φ, dφ];
* piece assignment: p ∈ γ_s belongs to piece π iff its foot on π's carrier lies within ε = 2h of π
  and |distance to the carrier| < 2h;
* effective density (averaged): A[p] = mean over the pieces of p of that piece's extension row;
  BEP rows: one per (p ∈ γ_in, π ∈ pieces(p)): E_π[p] - (P_γ A)[p], right-hand side Tr G f at p;
* the 8 row blocks are stacked into ONE least-squares problem (columns equilibrated to unit
  2-norm), solved exactly (numpy.linalg.lstsq), so every octant uses the same global C;
* PKS: each octant steps its own ρ̄, c with the global dt = min over octants of the
  Step-3 rule (R13); u_γ = A C clamped at 0 (R17); Green's formula per octant (R20);
* initial γ values (R31): average over the pieces of p of the piece's extension of the IC
  Cauchy data (cap: u0(foot); plane: u0(foot) + d ∂_a u0(foot)).

Parity unpinned vs the paper (the paper has no octant DD); pinned instead by a manufactured
zero-Neumann solution that the coupled DD solve reproduces at 2nd order, the 8-fold reflection
symmetry, and piece coverage (tests/test_oracle_dd.py).
"""
from dataclasses import dataclass, field
from typing import List

import numpy as np

from . import ap, dpm, grid, pks, sh

BOX = (-0.1, 1.1)   # canonical octant box (R3)
PIECES = ("cap", "x", "y", "z")


def octant_signs() -> List[np.ndarray]:
    """The 8 octants, index s = 4 [σx<0] + 2 [σy<0] + [σz<0]."""
    return [np.array([-1.0 if (s >> (2 - a)) & 1 else 1.0 for a in range(3)]) for s in range(8)]


def legendre(jmax: int, x: np.ndarray) -> np.ndarray:
    """P_0..P_jmax at x (Bonnet recurrence), shape (len(x), jmax+1)."""
    P = np.zeros((len(x), jmax + 1))
    P[:, 0] = 1.0
    if jmax >= 1:
        P[:, 1] = x
    for j in range(1, jmax):
        P[:, j + 1] = ((2 * j + 1) * x * P[:, j] - j * P[:, j - 1]) / (j + 1)
    return P


def plane_modes(Li: int):
    """(j, k) with j + k <= Li, ordered by total degree g then decreasing j."""
    return [(j, g - j) for g in range(Li + 1) for j in range(g, -1, -1)]


def plane_basis(Li: int, s: np.ndarray, t: np.ndarray) -> np.ndarray:
    Ps, Pt = legendre(Li, s), legendre(Li, t)
    return np.stack([Ps[:, j] * Pt[:, k] for j, k in plane_modes(Li)], axis=1)


def _dist_quarter_disc(s, t):
    """Euclidean distance from (s, t) to the quarter disc {s, t >= 0, s^2 + t^2 <= 1}."""
    ps, pt = np.maximum(s, 0.0), np.maximum(t, 0.0)
    r = np.hypot(ps, pt)
    scale = np.where(r > 1.0, 1.0 / np.where(r > 0, r, 1.0), 1.0)
    return np.hypot(s - ps * scale, t - pt * scale)


def _dist_octant_cap(f):
    """Distance from a point f on the unit sphere to the cap {|x| = 1, x >= 0}."""
    q = np.maximum(f, 0.0)
    nq = np.linalg.norm(q, axis=1, keepdims=True)
    q = q / np.where(nq > 0, nq, 1.0)
    return np.linalg.norm(f - q, axis=1)


@dataclass
class Octant:
    """One subdomain: canonical-frame grid and sets (shared), its signs and extension data."""
    s: int
    sigma: np.ndarray
    g: grid.Grid
    ps: grid.PointSets
    Eraw: np.ndarray          # |γ| × K: each piece's extension row (block-sparse by column)
    assign: np.ndarray        # |γ| × 4 bool: pieces of each γ point
    A: np.ndarray             # |γ| × K averaged effective density
    rows: np.ndarray          # (row_gamma_pos, piece) of the BEP rows: γ_in points x their pieces
    feet: dict = field(default_factory=dict)   # piece -> (|γ| × 3 physical foot, d)


@dataclass
class DDSetup:
    n: int
    Lc: int
    Li: int
    K: int
    blocks: dict              # piece -> column slice
    octants: List[Octant]


def column_blocks(Lc: int, Li: int):
    nc = (Lc + 1) ** 2
    nf = len(plane_modes(Li))
    blocks = {"cap": slice(0, 2 * nc)}
    for a, nm in enumerate("xyz"):
        blocks[nm] = slice(2 * nc + 2 * nf * a, 2 * nc + 2 * nf * (a + 1))
    return blocks, 2 * nc + 3 * 2 * nf


def piece_assignment(g: grid.Grid, ps: grid.PointSets) -> np.ndarray:
    """|γ| × 4 bool (cap, x, y, z): the foot on the piece's carrier lies within ε = 2h of the piece
    and |distance to the carrier| < 2h (R24; frame-independent, canonical octant)."""
    h = g.h
    eps = 2.0 * h
    P = dpm.gamma_points(g, ps)
    r = np.linalg.norm(P, axis=1)
    assign = np.zeros((len(P), 4), dtype=bool)
    assign[:, 0] = (_dist_octant_cap(P / r[:, None]) <= eps) & (np.abs(r - 1.0) < 2.0 * h)
    for a in range(3):
        o = [b for b in range(3) if b != a]
        assign[:, 1 + a] = (_dist_quarter_disc(P[:, o[0]], P[:, o[1]]) <= eps) & (np.abs(P[:, a]) < 2.0 * h)
    return assign


def setup(n: int, Lc: int, Li: int, which=None) -> DDSetup:
    """All 8 octants (which=None) or only the listed ones (the others are None: memory at n = 128)."""
    g = grid.Grid(n, *BOX)
    ps = grid.point_sets_from_mask(g, grid.octant_inside_mask(g))
    h = g.h
    eps = 2.0 * h
    P = dpm.gamma_points(g, ps)                        # canonical frame
    blocks, K = column_blocks(Lc, Li)
    nc = (Lc + 1) ** 2
    nf = len(plane_modes(Li))
    r = np.linalg.norm(P, axis=1)
    assign = piece_assignment(g, ps)
    gin_pos = np.searchsorted(ps.list("gamma"), ps.list("gamma_in"))
    rows = np.array([(q, k) for q in gin_pos for k in range(4) if assign[q, k]], dtype=np.int64).reshape(-1, 2)
    octs = []
    for s, sigma in enumerate(octant_signs()):
        if which is not None and s not in which:
            octs.append(None)
            continue
        E = np.zeros((len(P), K))
        X = sigma * P                                  # physical coordinates
        # cap: foot on the unit sphere, d = |x| - 1 (+ outside), zero Neumann -> {Y, d^2/2 Y}
        Y = sh.real_sh(Lc, X / r[:, None])
        dcap = r - 1.0
        E[:, blocks["cap"]] = np.concatenate([Y, 0.5 * (dcap ** 2)[:, None] * Y], axis=1)
        feet = {"cap": (X / r[:, None], dcap)}
        for a, nm in enumerate("xyz"):
            o = [b for b in range(3) if b != a]
            phi = plane_basis(Li, X[:, o[0]], X[:, o[1]])
            d = X[:, a]                                # signed distance along +e_a (R25)
            E[:, blocks[nm]] = np.concatenate([phi, d[:, None] * phi], axis=1)
            foot = X.copy()
            foot[:, a] = 0.0
            feet[nm] = (foot, d)
        cnt = assign.sum(axis=1)
        mask = np.zeros((len(P), K))
        for k, nm in enumerate(PIECES):
            mask[:, blocks[nm]] = assign[:, k:k + 1]
        A = E * mask / np.maximum(cnt, 1)[:, None]
        octs.append(Octant(s, sigma, g, ps, E, assign, A, rows, feet))
    assert nc > 0 and nf > 0
    return DDSetup(n, Lc, Li, K, blocks, octs)


def bep_block(st: DDSetup, o: Octant, dt: float):
    """Rows E_π[p] - (P_γ A)[p] for (p, π) in o.rows, and the potential columns' γ trace."""
    PgA = dpm.potential_trace(o.A, o.g, o.ps, dt, o.ps.list("gamma"))   # K AP solves, |γ| × K
    B = np.zeros((len(o.rows), st.K))
    for i, (q, k) in enumerate(o.rows):
        blk = st.blocks[PIECES[k]]
        B[i, blk] = o.Eraw[q, blk]
        B[i] -= PgA[q]
    return B, PgA


def stacked_lstsq(Bs: List[np.ndarray], gs: List[np.ndarray]) -> np.ndarray:
    """Global C = argmin || [B_s] C - [g_s] ||, columns equilibrated to unit 2-norm (R24)."""
    Bst = np.concatenate(Bs, axis=0)
    gst = np.concatenate(gs, axis=0)
    D = 1.0 / np.linalg.norm(Bst, axis=0)
    return D[:, None] * np.linalg.lstsq(Bst * D, gst, rcond=None)[0] if gst.ndim > 1 else \
        D * np.linalg.lstsq(Bst * D, gst, rcond=None)[0]


def coupled_solve(st: DDSetup, f_boxes, dt: float, Bs=None):
    """One coupled DPM solve of (I/dt - Δ_h) u = f/dt on every octant (R4 scaling as PKS uses):
    particular solutions, the stacked BEP LSQ, u_γ = A C, Green's formula per octant."""
    if Bs is None:
        Bs = [bep_block(st, o, dt)[0] for o in st.octants]
    gs = []
    for o, f in zip(st.octants, f_boxes):
        up = ap.solve(dpm.particular_rhs(f, o.ps, dt), o.g.h, dt)
        gvec = dpm.trace(up, o.ps.list("gamma"))
        gs.append(gvec[o.rows[:, 0]])
    C = stacked_lstsq(Bs, gs)
    us = [dpm.green(o.A @ C, f, o.g, o.ps, dt) for o, f in zip(st.octants, f_boxes)]
    return us, C, Bs


def ic_fields(st: DDSetup, center, rho_ic, c_ic):
    """R14 / R31: IC at the node on N+ (physical coordinates); on γ the average over the point's
    pieces of the piece's extension of the IC Cauchy data."""
    c0 = np.asarray(center, dtype=float)
    out = []
    for o in st.octants:
        x = o.g.coords()
        Xc, Yc, Zc = np.meshgrid(x, x, x, indexing="ij")
        Xp = np.stack([Xc, Yc, Zc], axis=-1) * o.sigma

        def gauss(A, a, X):
            return A * np.exp(-a * ((X - c0) ** 2).sum(axis=-1))

        def dgauss(A, a, X, ax):
            return -2.0 * a * (X[..., ax] - c0[ax]) * gauss(A, a, X)

        fields = []
        for (Am, am) in (rho_ic, c_ic):
            F = np.where(o.ps.nplus, gauss(Am, am, Xp), 0.0)
            gidx = o.ps.list("gamma")
            acc = np.zeros(len(gidx))
            for k, nm in enumerate(PIECES):
                foot, d = o.feet[nm]
                val = gauss(Am, am, foot)
                if nm != "cap":
                    val = val + d * dgauss(Am, am, foot, "xyz".index(nm))
                acc += np.where(o.assign[:, k], val, 0.0)
            F.reshape(-1)[gidx] = acc / np.maximum(o.assign.sum(axis=1), 1)
            fields.append(F)
        out.append(tuple(fields))
    return out


class DDPKSOracle:
    """PKS time stepping (Steps 1-8) on the 8 coupled octants (R24, R13-R20, R31)."""

    def __init__(self, n, Lc, Li, dt_cap, steps, chi=1.0, center=(0.0, 0.0, 0.0),
                 rho_ic=(1000.0, 100.0), c_ic=(500.0, 50.0), clamp=True):
        self.st = setup(n, Lc, Li)
        self.dt_cap, self.steps, self.chi = dt_cap, steps, chi
        self.center, self.rho_ic, self.c_ic, self.clamp = center, rho_ic, c_ic, clamp
        self.dt_prev = np.inf
        self.dt_bep = None
        self.Bs = None
        self.builds = 0
        self.t = 0.0

    def initial_state(self):
        return ic_fields(self.st, self.center, self.rho_ic, self.c_ic)

    def step(self, state):
        st, chi = self.st, self.chi
        h = st.octants[0].g.h
        dts = [pks.cfl_dt(c, o.ps, h, chi) for o, (_, c) in zip(st.octants, state)]
        dt = min(self.dt_prev, self.dt_cap, min(dts), 0.5 * h * h)      # Step 3 + R13, global min (C4)
        rebuilt = False
        if self.Bs is None or dt != self.dt_bep:                          # Step 2 / 4b
            self.Bs = [bep_block(st, o, dt)[0] for o in st.octants]
            self.dt_bep = dt
            self.builds += 1
            rebuilt = True
        new = [[None, None] for _ in st.octants]
        frhs = []
        for o, (rho, c) in zip(st.octants, state):
            gconv = pks.convection(rho, c, o.ps, h, chi)
            frhs.append(pks.assemble_rhs(rho, c, gconv, dt))                 # Step 4a
        for fi in range(2):
            fs, gvecs = [], []
            for o, fr in zip(st.octants, frhs):
                f = fr[fi]
                up = ap.solve(dpm.particular_rhs(f, o.ps, dt), h, dt)
                gvecs.append(dpm.trace(up, o.ps.list("gamma"))[o.rows[:, 0]])
                fs.append(f)
            C = stacked_lstsq(self.Bs, gvecs)                                 # Step 5 (global)
            for s, (o, f) in enumerate(zip(st.octants, fs)):
                ug = o.A @ C
                if self.clamp:
                    ug = np.maximum(ug, 0.0)                              # R17
                new[s][fi] = dpm.green(ug, f, o.g, o.ps, dt)              # Steps 6-7 (R20)
        self.dt_prev = dt
        self.t += dt
        return [tuple(x) for x in new], dict(dt=dt, rebuilt=rebuilt, t=self.t)

    def mass(self, state):
        h = self.st.octants[0].g.h
        return h ** 3 * sum(rho[o.ps.mplus].sum() for o, (rho, _) in zip(self.st.octants, state))

    def run(self, nsteps=None):
        state = self.initial_state()
        logs = []
        for _ in range(nsteps if nsteps is not None else self.steps):
            state, log = self.step(state)
            log["mass"] = self.mass(state)
            logs.append(log)
        return state, logs


# ---- config 5 at its configured size through the exact 8-fold reflection symmetry -----------------
# The octants share the canonical-frame grid, sets, pieces and rows; octant s's extension is octant 0's
# with column signs, E_s = E_0 diag(S_s) (real SH and Legendre products are even or odd under each
# reflection x_a -> -x_a, and d = x_a on the planes flips with σ_a), hence A_s = A_0 diag(S_s) and
# B_s = B_0 diag(S_s).  For an IC symmetric under all 8 reflections (cfg5: centred at the origin) every
# octant's canonical state is the same, so g_s = g_0 and the stacked least squares
#     min_C Σ_s || B_0 S_s C - g_0 ||^2
# is the one of `stacked_lstsq`.  With B_0 = Q R (thin QR) each term is || R S_s C - Q^T g_0 ||^2 plus a
# constant, so the (8K x K) system [R S_s]_s C = [Q^T g_0]_s has the same minimiser (SURVEY probe P9/P12
# used the same reduction).  Its column norms are those of the stacked matrix (= sqrt(8) |B_0[:, c]|).

def column_signs(st: DDSetup, sigmas=None) -> np.ndarray:
    """(8, K) S_s with E_s = E_0 diag(S_s), read off the extension of octant 0's γ points under each σ
    (asserted to be exactly ±1 on every column)."""
    o0 = st.octants[0]
    P = dpm.gamma_points(o0.g, o0.ps)
    P = P[:: max(1, len(P) // 4000)]        # a few thousand γ points determine every column's sign
    blocks = st.blocks
    out = np.ones((8, st.K))
    r = np.linalg.norm(P, axis=1)
    def ext(sig):
        X = sig * P
        Y = sh.real_sh(st.Lc, X / r[:, None])
        cols = [Y, 0.5 * ((r - 1.0) ** 2)[:, None] * Y]
        for a in range(3):
            o = [b for b in range(3) if b != a]
            phi = plane_basis(st.Li, X[:, o[0]], X[:, o[1]])
            cols += [phi, X[:, a][:, None] * phi]
        return np.concatenate(cols, axis=1)
    E0 = ext(octant_signs()[0])
    q = np.argmax(np.abs(E0), axis=0)
    for s, sig in enumerate(octant_signs()):
        Es = ext(sig)
        ratio = Es[q, np.arange(st.K)] / E0[q, np.arange(st.K)]
        assert np.allclose(np.abs(ratio), 1.0, rtol=1e-12, atol=0), "extension not ±1 under reflection"
        assert np.allclose(Es, E0 * np.sign(ratio), rtol=0, atol=1e-13 * np.abs(E0).max())
        out[s] = np.sign(ratio)
    assert len(blocks) == 4
    return out


def stacked_lstsq_symmetric(B0: np.ndarray, signs: np.ndarray, g0: np.ndarray) -> np.ndarray:
    """`stacked_lstsq` of the blocks B_0 diag(S_s) with the common right-hand side g_0, through the
    thin QR of B_0 (see the block comment above); g0 may hold several columns."""
    Q, R = np.linalg.qr(B0)
    z = Q.T @ g0
    Bst = np.concatenate([R * s for s in signs], axis=0)                 # R S_s
    zst = np.concatenate([z] * len(signs), axis=0)
    D = 1.0 / np.linalg.norm(Bst, axis=0)
    y = np.linalg.lstsq(Bst * D, zst, rcond=None)[0]
    return (D[:, None] * y) if y.ndim > 1 else D * y


class DDPKSOracleSymmetric(DDPKSOracle):
    """DDPKSOracle for an IC symmetric under the 8 reflections, simulating octant 0 only (every octant's
    canonical state is the same): the global dt is octant 0's rule, the global C the symmetric stacked
    least squares.  Same steps and readings as DDPKSOracle.step, one octant's arithmetic."""

    def __init__(self, n, Lc, Li, dt_cap, steps, **kw):
        self.st = setup(n, Lc, Li, which=(0,))
        self.signs = column_signs(self.st)
        self.dt_cap, self.steps = dt_cap, steps
        self.chi = kw.get("chi", 1.0)
        self.center = kw.get("center", (0.0, 0.0, 0.0))
        assert all(c == 0.0 for c in self.center), "the reduction needs an origin-centred (symmetric) IC"
        self.rho_ic, self.c_ic = kw.get("rho_ic", (1000.0, 100.0)), kw.get("c_ic", (500.0, 50.0))
        self.clamp = kw.get("clamp", True)
        self.dt_prev, self.dt_bep, self.B0, self.builds, self.t = np.inf, None, None, 0, 0.0

    def initial_state(self):
        st = self.st
        full = DDSetup(st.n, st.Lc, st.Li, st.K, st.blocks, [st.octants[0]])
        return ic_fields(full, self.center, self.rho_ic, self.c_ic)[0]

    def step(self, state):
        o = self.st.octants[0]
        h, chi = o.g.h, self.chi
        rho, c = state
        dt = min(self.dt_prev, self.dt_cap, pks.cfl_dt(c, o.ps, h, chi), 0.5 * h * h)   # Step 3 + R13
        rebuilt = False
        if self.B0 is None or dt != self.dt_bep:                                       # Step 2 / 4b
            self.B0 = bep_block(self.st, o, dt)[0]
            self.dt_bep = dt
            self.builds += 1
            rebuilt = True
        gconv = pks.convection(rho, c, o.ps, h, chi)
        frhs = pks.assemble_rhs(rho, c, gconv, dt)                                      # Step 4a
        new = []
        for f in frhs:
            up = ap.solve(dpm.particular_rhs(f, o.ps, dt), h, dt)
            g0 = dpm.trace(up, o.ps.list("gamma"))[o.rows[:, 0]]
            C = stacked_lstsq_symmetric(self.B0, self.signs, g0)                        # Step 5 (global)
            ug = o.A @ C
            if self.clamp:
                ug = np.maximum(ug, 0.0)                                                # R17
            new.append(dpm.green(ug, f, o.g, o.ps, dt))                                 # Steps 6-7 (R20)
        self.dt_prev = dt
        self.t += dt
        return tuple(new), dict(dt=dt, rebuilt=rebuilt, t=self.t)

    def mass(self, state):
        o = self.st.octants[0]
        return 8 * o.g.h ** 3 * state[0][o.ps.mplus].sum()
