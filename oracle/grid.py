"""Grid and point sets — oracle (test infrastructure only).

Grid: the cube [lo, hi]^3 has its faces on the Dirichlet (ghost)
layer N0 \\ M0; ``n`` unknowns per axis, h = (hi - lo)/(n + 1), node
i (0-based, 0..n-1) at lo + (i + 1) h.  The full lattice N0 is (n+2)^3 with
lattice index i+1 for node i, ghosts at lattice indices 0 and n+1.

Point sets: Definition 1, literally, as set algebra on the lattice:
  M0 = interior nodes; M+ = M0 ∩ Ω (open interior, ties -> M-, R6);
  M- = M0 \\ M+;  N± = union of 7-point stencils of M±;
  gamma = N+ ∩ N-;  gamma_in = M+ ∩ gamma;  gamma_ex = M- ∩ gamma.
Lists are ascending flat indices of the C-order [x][y][z] interior (R7).
"band" = M- ∩ dil7(gamma): the support of any difference-potential RHS (R21).

Classification is EXACT (R6): coordinates are rationals built from the decimal
reading of the configuration numbers and the inside test is evaluated in exact
integer arithmetic.
"""
from dataclasses import dataclass
from fractions import Fraction
from functools import reduce
from math import gcd

import numpy as np


@dataclass
class Grid:
    n: int
    lo: float
    hi: float

    @property
    def h(self) -> float:
        return (self.hi - self.lo) / (self.n + 1)

    def coords(self) -> np.ndarray:
        """Node coordinates x_i = lo + (i+1) h, i = 0..n-1 (R1)."""
        return self.lo + (np.arange(self.n) + 1.0) * self.h


def _frac(x: float) -> Fraction:
    # decimal reading of the configuration constant (e.g. -1.1 -> -11/10)
    return Fraction(repr(float(x)))


def _lcm(a: int, b: int) -> int:
    return a * b // gcd(a, b)


def inside_mask(grid: Grid, kind: str, center, semi) -> np.ndarray:
    """Boolean [n][n][n]: node strictly inside Ω (M+ membership), exact rationals.

    sphere / ellipsoid: sum_a ((x_a - c_a)/s_a)^2 < 1 (P:596 sphere; R10 ellipsoid).
    Ties (== 1) go to M- (R6).
    """
    n = grid.n
    lo, hi = _frac(grid.lo), _frac(grid.hi)
    terms = []
    for a in range(3):
        c, s = _frac(center[a]), _frac(semi[a])
        vals = [((lo + (i + 1) * (hi - lo) / (n + 1)) - c) ** 2 / s ** 2 for i in range(n)]
        terms.append(vals)
    den = reduce(_lcm, [v.denominator for t in terms for v in t], 1)
    ints = [np.array([int(v * den) for v in t], dtype=object) for t in terms]
    tot = ints[0][:, None, None] + ints[1][None, :, None] + ints[2][None, None, :]
    return np.asarray(tot < den, dtype=bool)


def shell_inside_mask(grid: Grid, r_in, r_out, center=(0.0, 0.0, 0.0)) -> np.ndarray:
    """Boolean [n][n][n]: node strictly inside the spherical shell r_in < |x - c| < r_out (the outer
    subdomain Ω2 of the paper's concentric domain decomposition, Case 1), exact
    rationals; nodes on either sphere go to M- (R6)."""
    n = grid.n
    lo, hi = _frac(grid.lo), _frac(grid.hi)
    terms = []
    for a in range(3):
        c = _frac(center[a])
        terms.append([((lo + (i + 1) * (hi - lo) / (n + 1)) - c) ** 2 for i in range(n)])
    ri, ro = _frac(r_in) ** 2, _frac(r_out) ** 2
    den = reduce(_lcm, [v.denominator for t in terms for v in t] + [ri.denominator, ro.denominator], 1)
    ints = [np.array([int(v * den) for v in t], dtype=object) for t in terms]
    tot = ints[0][:, None, None] + ints[1][None, :, None] + ints[2][None, None, :]
    return np.asarray((tot > int(ri * den)) & (tot < int(ro * den)), dtype=bool)


def _dilate7(mask_lat: np.ndarray) -> np.ndarray:
    """Union of 7-point stencils of the True points, within the lattice."""
    out = mask_lat.copy()
    for ax in range(3):
        for sgn in (1, -1):
            sh = np.zeros_like(mask_lat)
            src = [slice(None)] * 3
            dst = [slice(None)] * 3
            if sgn == 1:
                src[ax] = slice(0, -1)
                dst[ax] = slice(1, None)
            else:
                src[ax] = slice(1, None)
                dst[ax] = slice(0, -1)
            sh[tuple(dst)] = mask_lat[tuple(src)]
            out |= sh
    return out


@dataclass
class PointSets:
    n: int
    mplus: np.ndarray        # bool [n][n][n]
    nplus_lat: np.ndarray    # bool [n+2]^3 (lattice incl. ghosts)
    nminus_lat: np.ndarray
    gamma: np.ndarray        # bool [n][n][n]
    gamma_in: np.ndarray
    gamma_ex: np.ndarray
    band: np.ndarray

    @property
    def nplus(self) -> np.ndarray:
        """N+ restricted to the interior M0."""
        return self.nplus_lat[1:-1, 1:-1, 1:-1]

    @property
    def ghosts_in_nplus(self) -> int:
        return int(self.nplus_lat.sum() - self.nplus.sum())

    def list(self, which: str) -> np.ndarray:
        m = {"mplus": self.mplus, "gamma": self.gamma, "gamma_in": self.gamma_in,
             "gamma_ex": self.gamma_ex, "band": self.band, "nplus": self.nplus,
             "mminus": ~self.mplus}[which]
        return np.flatnonzero(m.ravel()).astype(np.int64)


def octant_inside_mask(grid: Grid, radius=1.0) -> np.ndarray:
    """cfg5 subdomain in its canonical frame: the open octant
    {x, y, z > 0} ∩ {|x| < radius}, exact rationals; nodes on a plane or on the sphere go to M-."""
    n = grid.n
    lo, hi, r = _frac(grid.lo), _frac(grid.hi), _frac(radius)
    xs = [lo + (i + 1) * (hi - lo) / (n + 1) for i in range(n)]
    den = reduce(_lcm, [v.denominator for v in xs] + [r.denominator], 1)
    X = np.array([int(v * den) for v in xs], dtype=object)
    pos = X > 0
    sq = X * X
    tot = sq[:, None, None] + sq[None, :, None] + sq[None, None, :]
    inside = np.asarray(tot < int(r * den) ** 2, dtype=bool)
    return inside & pos[:, None, None] & pos[None, :, None] & pos[None, None, :]


def point_sets(grid: Grid, kind: str, center, semi) -> PointSets:
    """Definition 1 on the (n+2)^3 lattice N0 including the ghost layer (R5)."""
    return point_sets_from_mask(grid, inside_mask(grid, kind, center, semi))


def point_sets_from_mask(grid: Grid, mplus: np.ndarray) -> PointSets:
    """Definition 1 for a given M+ mask."""
    n = grid.n
    lat = np.zeros((n + 2,) * 3, dtype=bool)
    mp_lat = lat.copy()
    mp_lat[1:-1, 1:-1, 1:-1] = mplus
    mm_lat = lat.copy()
    mm_lat[1:-1, 1:-1, 1:-1] = ~mplus
    np_lat = _dilate7(mp_lat)       # N+ = ∪ stencils of M+
    nm_lat = _dilate7(mm_lat)       # N- = ∪ stencils of M-
    gam_lat = np_lat & nm_lat       # gamma = N+ ∩ N-
    gamma = gam_lat[1:-1, 1:-1, 1:-1].copy()
    assert gam_lat.sum() == gamma.sum(), "a ghost node cannot be in gamma (R5)"
    gamma_in = mplus & gamma
    gamma_ex = (~mplus) & gamma
    band = (~mplus) & _dilate7(gam_lat)[1:-1, 1:-1, 1:-1]
    return PointSets(n, mplus, np_lat, nm_lat, gamma, gamma_in, gamma_ex, band)


def point_sets_for(cfg) -> "tuple[Grid, PointSets]":
    g = Grid(cfg.n, cfg.lo, cfg.hi)
    return g, point_sets(g, cfg.kind, cfg.center, cfg.semi)
