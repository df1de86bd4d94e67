"""Pins for oracle/grid.py: Definition 1 point sets and exact classification (R6)."""
import json
import os

import numpy as np
import pytest

from dpm_inputs import get_config
from oracle import grid

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "point_set_counts.json")


def brute_force_sets(n, inside):
    """Def. 1 by explicit loops over the (n+2)^3 lattice and 7-point stencils."""
    M = {}
    for i in range(n):
        for j in range(n):
            for k in range(n):
                M[(i, j, k)] = inside(i, j, k)
    stencil = [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]
    Np, Nm = set(), set()
    for p, ins in M.items():
        for s in stencil:
            q = (p[0] + s[0], p[1] + s[1], p[2] + s[2])
            (Np if ins else Nm).add(q)
    gamma = Np & Nm
    flat = lambda q: (q[0] * n + q[1]) * n + q[2]
    gam = sorted(flat(q) for q in gamma)
    gin = sorted(flat(q) for q in gamma if M.get(q, False))
    gex = sorted(flat(q) for q in gamma if q in M and not M[q])
    ghosts = sum(1 for q in Np if q not in M)
    return gam, gin, gex, ghosts


@pytest.mark.parametrize("n", [12, 16])
def test_sphere_sets_brute_force_integer(n):
    # R6: for the unit sphere in [-1.1,1.1]^3, x_i = 1.1 X/(n+1) with X = 2i-n+1, so
    # inside <=> 121 (X^2+Y^2+Z^2) < 100 (n+1)^2 (exact integers, independent of oracle).
    def inside(i, j, k):
        X, Y, Z = 2 * i - n + 1, 2 * j - n + 1, 2 * k - n + 1
        return 121 * (X * X + Y * Y + Z * Z) < 100 * (n + 1) ** 2

    gam, gin, gex, ghosts = brute_force_sets(n, inside)
    g = grid.Grid(n, -1.1, 1.1)
    ps = grid.point_sets(g, "sphere", (0, 0, 0), (1, 1, 1))
    assert list(ps.list("gamma")) == gam
    assert list(ps.list("gamma_in")) == gin
    assert list(ps.list("gamma_ex")) == gex
    assert ps.ghosts_in_nplus == ghosts


def test_ellipsoid_integer_formula_cfg3():
    # R6: ellipsoid (0.9,0.6,0.5) in [-1,1]^3: 100X^2 + 225Y^2 + 324Z^2 < 81 (n+1)^2.
    cfg = get_config("cfg3")
    n = cfg.n
    X = 2 * np.arange(n) - n + 1
    ref = (100 * X[:, None, None] ** 2 + 225 * X[None, :, None] ** 2 + 324 * X[None, None, :] ** 2
           < 81 * (n + 1) ** 2)
    g = grid.Grid(n, cfg.lo, cfg.hi)
    assert np.array_equal(grid.inside_mask(g, cfg.kind, cfg.center, cfg.semi), ref)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4"])
def test_counts_golden(name):
    fx = json.load(open(GOLDEN))[name]
    g, ps = grid.point_sets_for(get_config(name))
    got = {"mplus": int(ps.mplus.sum()), "gamma": int(ps.gamma.sum()), "gamma_in": int(ps.gamma_in.sum()),
           "gamma_ex": int(ps.gamma_ex.sum()), "ghosts_in_nplus": ps.ghosts_in_nplus, "band": int(ps.band.sum())}
    assert got == fx


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_set_invariants(name):
    g, ps = grid.point_sets_for(get_config(name))
    assert not (ps.gamma_in & ps.gamma_ex).any()
    assert np.array_equal(ps.gamma_in | ps.gamma_ex, ps.gamma)
    # every N+ \ M+ interior point is in gamma (Def. 1 consequence)
    assert not (ps.nplus & ~ps.mplus & ~ps.gamma).any()
    # the band is in M- and contains gamma_ex
    assert not (ps.band & ps.mplus).any()
    assert not (ps.gamma_ex & ~ps.band).any()


def test_gamma_scaling():
    # |gamma| = O(h^-2): ratio |γ(N)|/|γ(2N)| in [0.2, 0.35]
    sizes = []
    for n in (20, 40):
        g = grid.Grid(n, -1.1, 1.1)
        sizes.append(grid.point_sets(g, "sphere", (0, 0, 0), (1, 1, 1)).gamma.sum())
    assert 0.2 <= sizes[0] / sizes[1] <= 0.35


@pytest.mark.parametrize("N", [36, 68, 132])
def test_paper_mesh_point_sets(N):
    # the paper's mesh convention through dpm_inputs.paper_mesh: h = 2r/(N-4), cell centres at
    # -r + (j - 5/2) h, against the survey's independent exact-integer counts (probe P1)
    from dpm_inputs import paper_mesh
    n, lo, hi, h = paper_mesh(N, 0.5)
    assert n == N and abs(h - 1.0 / (N - 4)) < 1e-16
    g = grid.Grid(n, lo, hi)
    assert abs(g.h - h) < 1e-15
    x = g.coords()
    assert np.allclose(x, -0.5 + (np.arange(1, N + 1) - 2.5) * h, atol=1e-14)
    ps = grid.point_sets(g, "sphere", (0.0, 0.0, 0.0), (0.5, 0.5, 0.5))
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "point_set_counts.json")))["paper_meshes"][str(N)]
    assert len(ps.list("gamma")) == ref["gamma"]
    assert len(ps.list("gamma_in")) == ref["gamma_in"]


def _exact_ties_sphere(n):
    # nodes exactly on the unit sphere in [-1.1, 1.1]^3 (R6 closed form: 121 (X²+Y²+Z²) = 100 (n+1)²,
    # X = 2i - n + 1), counted by brute force over integer triples
    X = 2 * np.arange(n) - n + 1
    s = (X[:, None, None] ** 2 + X[None, :, None] ** 2 + X[None, None, :] ** 2) * 121
    return int((s == 100 * (n + 1) ** 2).sum())


@pytest.mark.parametrize("n,ties", [(65, 150), (16, 0), (32, 0), (128, 0)])
def test_sphere_tie_meshes_and_rule(n, ties):
    # R6 ties -> M-: the advisor's n = 65 mesh has nodes exactly on Γ (the GPU tie test uses it); the
    # configured meshes have none.  The oracle's exact classification puts every tie in M-.
    assert _exact_ties_sphere(n) == ties
    if ties:
        g = grid.Grid(n, -1.1, 1.1)
        m = grid.inside_mask(g, "sphere", (0.0, 0.0, 0.0), (1.0, 1.0, 1.0))
        X = 2 * np.arange(n) - n + 1
        s = (X[:, None, None] ** 2 + X[None, :, None] ** 2 + X[None, None, :] ** 2) * 121
        assert not m[s == 100 * (n + 1) ** 2].any()
        assert np.array_equal(m, s < 100 * (n + 1) ** 2)
