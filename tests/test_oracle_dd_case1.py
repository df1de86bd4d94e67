"""Pins of the two-subdomain Case-1 DD oracle (oracle/dd_case1.py).

* Reduction to the single domain: one subdomain = the whole ball with only the Γ piece is exactly the
  single-domain method (same extension columns, reduced BEP and PKS step as oracle/dpm.py, oracle/pks.py
  with the paper's zonal 3-term zero-Neumann basis).
* Manufactured solution across Z: a smooth u* on Ω with ∂_r u* = 0 on Γ; the coupled BEPs with the
  shared interface Cauchy data reproduce it in BOTH subdomains at second order in h (P:549 remark (i)).
* Point sets: Ω1 ∪ Ω2 cover the ball's interior nodes of each mesh exactly once where the meshes
  coincide (N1 = 2 N2 - 4 nests h1 = h2 / ... only on the common mesh, tested for h1 = h2 / 2 below).
"""
import numpy as np
import pytest

from dpm_inputs import paper_mesh
from dpm_inputs import test_a_config as sd_config
from oracle import ap, dd_case1 as dc, dpm, grid, pks


def test_extension_blocks_and_pieces():
    dd = dc.CaseOneDD(20, 20, 1e-8, 1)
    ball, shell = dd.subs
    zb, gb, K = dc.column_blocks(0, 0)
    assert K == 5 and dd.K == 5
    assert np.all(ball.piece == dc.Z_PIECE)
    rad = np.sqrt((dpm.gamma_points(shell.g, shell.ps) ** 2).sum(axis=1))
    # the two layers of Ω2's discrete boundary sit within 2 h2 of their spheres
    h2 = shell.g.h
    assert np.all(np.abs(rad[shell.piece == dc.Z_PIECE] - 0.25) < 2 * h2)
    assert np.all(np.abs(rad[shell.piece == dc.G_PIECE] - 0.5) < 2 * h2)
    assert (shell.piece == dc.Z_PIECE).sum() > 0 and (shell.piece == dc.G_PIECE).sum() > 0
    # Z rows carry u, d u, d²/2 u with d = |x| - r1; Γ rows u, d²/2 u with d = |x| - r2; nothing else
    for s in (ball, shell):
        z = s.piece == dc.Z_PIECE
        assert np.all(s.E[z][:, gb] == 0) and np.all(s.E[~z][:, zb] == 0)
        assert np.allclose(s.E[z][:, 0], 1.0) and np.allclose(s.E[z][:, 1], s.d[z])
        assert np.allclose(s.E[z][:, 2], 0.5 * s.d[z] ** 2)
        if (~z).any():
            assert np.allclose(s.E[~z][:, 3], 1.0) and np.allclose(s.E[~z][:, 4], 0.5 * s.d[~z] ** 2)


def test_meshes_are_the_papers():
    # N_l cells, h_l = 2 r_l / (N_l - 4); 20/20 gives h1 = 1/32 (= the SD N = 36 mesh)
    dd = dc.CaseOneDD(20, 20, 1e-8, 1)
    assert abs(dd.subs[0].g.h - 1 / 32) < 1e-15 and abs(dd.subs[1].g.h - 1 / 16) < 1e-15
    assert abs(dd.subs[0].g.h - paper_mesh(36, 0.5)[3]) < 1e-15


def _single_domain_as_dd(N):
    # the whole ball r = 0.5 treated as one Case-1 subdomain whose boundary is all Γ
    cfg = sd_config(N)
    n, lo, hi, _ = paper_mesh(N, 0.5)
    g = grid.Grid(n, lo, hi)
    ps = grid.point_sets(g, "sphere", (0.0, 0.0, 0.0), (0.5, 0.5, 0.5))
    P = dpm.gamma_points(g, ps)
    piece = np.full(len(P), dc.G_PIECE)
    E, foot, d = dc.extension_rows(P, piece, 0.25, 0.5, 0, 0)
    sub = dc.Subdomain("ball", g, ps, piece, E, foot, d,
                       np.searchsorted(ps.list("gamma"), ps.list("gamma_in")))
    return cfg, sub


def test_single_subdomain_reduces_to_the_single_domain_method():
    cfg, sub = _single_domain_as_dd(36)
    g, ps = grid.point_sets_for(cfg)
    Esd, _, _, _ = dpm.extension_matrix(g, ps, cfg.kind, cfg.center, cfg.semi, cfg.lmax, cfg.basis)
    assert np.abs(sub.E[:, 3:] - Esd).max() <= 1e-15
    dt = 1e-8
    B = dc.bep_rows(sub, dt)
    _, Bsd, _ = dpm.projection_and_bep(Esd, g, ps, dt)
    assert np.abs(B[:, 3:] - Bsd).max() <= 1e-12 * np.abs(Bsd).max()
    # one PKS step of the DD machinery with this single subdomain = the single-domain oracle's step
    dd = dc.CaseOneDD(20, 20, dt, 1, dt_rule=1)
    dd.subs = [sub]
    dd.K = 5
    dd.Bs = [B[:, 3:]]
    dd.dt_bep = dt
    for s in dd.subs:
        s.E = s.E[:, 3:]
    state = dd.initial_state()
    o = pks.PKSOracle(cfg, dt_rule=1)
    r0, c0 = o.initial_state()
    assert np.abs(state[0][0] - r0).max() <= 1e-12 * np.abs(r0).max()
    assert np.abs(state[0][1] - c0).max() <= 1e-12 * np.abs(c0).max()
    (rho, c), = dd.step(state)[0]
    ro, co, _ = o.step(r0, c0)
    assert np.abs(rho - ro).max() <= 1e-11 * np.abs(ro).max()
    assert np.abs(c - co).max() <= 1e-11 * np.abs(co).max()


def mms_errors(N1, N2, dt=1e-2, M=2):
    """u* = cos(2π r) + z (1 - 4 r²/3): smooth on Ω, ∂_r u* = 0 at r = 0.5; Δu* = -4π² cos(2πr)
    - (4π/r) sin(2πr) - 40 z / 3.  f = (I - dt Δ) u* on each subdomain; max error over M_l+."""
    dd = dc.CaseOneDD(N1, N2, dt, 1, Mz=M, Mg=M)
    fs, us = [], []
    for s in dd.subs:
        x = s.g.coords()
        X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
        R = np.sqrt(X ** 2 + Y ** 2 + Z ** 2)
        u = np.cos(2 * np.pi * R) + Z * (1 - 4 * R ** 2 / 3)
        lap = -4 * np.pi ** 2 * np.cos(2 * np.pi * R) - 4 * np.pi * np.sin(2 * np.pi * R) / R - 40 * Z / 3
        fs.append(u - dt * lap)
        us.append(u)
    sol, _ = dc.coupled_elliptic_solve(dd, fs, dt)
    return [np.abs(v - u)[s.ps.mplus].max() for v, u, s in zip(sol, us, dd.subs)]


@pytest.mark.slow
def test_manufactured_solution_across_the_interface_second_order():
    e1 = mms_errors(20, 20)
    e2 = mms_errors(36, 36)
    for a, b in zip(e1, e2):
        assert 3.0 < a / b < 5.5, (e1, e2)        # h halves: second order in both subdomains
    assert max(e2) < 5e-3
