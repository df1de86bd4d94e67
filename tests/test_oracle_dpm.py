"""Pins for oracle/dpm.py: projections, BEP theorems, LSQ, Green's formula."""
import numpy as np
import pytest

from dpm_inputs import get_config
from dpm_inputs.rng import uniform_values
from oracle import ap, dpm, grid


@pytest.fixture(scope="module")
def cfg1_proj():
    cfg = get_config("cfg1")
    g, ps = grid.point_sets_for(cfg)
    return cfg, g, ps, dpm.full_projection(g, ps, cfg.dt)


def test_projection_idempotent(cfg1_proj):
    # P_γ is a projection
    cfg, g, ps, P = cfg1_proj
    assert np.abs(P @ P - P).max() / np.abs(P).max() < 1e-12


def test_rank_prop1(cfg1_proj):
    # Prop. 1: rank of the BEP (I - P_γ) = |γ_in|
    cfg, g, ps, P = cfg1_proj
    s = np.linalg.svd(np.eye(len(P)) - P, compute_uv=False)
    r = int(ps.gamma_in.sum())
    assert (s > 1e-8).sum() == r
    assert s[r - 1] > 0.5 and s[r] < 1e-12


def test_thm1_and_green_reproduce_difference_solution(cfg1_proj):
    # Thm 1 + Green: for ANY grid function u on N+ (0 on ghosts),
    # with f = L u on M+, the trace u_γ satisfies u_γ - P_γ u_γ = Tr_γ G f and
    # P_{N+γ} u_γ + G f = u on N+.
    cfg, g, ps, P = cfg1_proj
    n, dt = g.n, cfg.dt
    u = np.where(ps.nplus, uniform_values(11, (n, n, n)), 0.0)
    f_paper = dt * ap.apply_operator(u, g.h, dt)          # L = I - dt Δ_h = dt (I/dt - Δ_h)
    gidx = ps.list("gamma")
    u_g = u.reshape(-1)[gidx]
    Gf = ap.solve(dpm.particular_rhs(f_paper, ps, dt), g.h, dt).reshape(-1)[gidx]
    assert np.abs(u_g - P @ u_g - Gf).max() < 1e-12
    rec = dpm.green(u_g, f_paper, g, ps, dt)
    assert np.abs(rec - u).max() < 1e-12
    rec2 = dpm.green_two_solve(u_g, f_paper, g, ps, dt)
    assert np.abs(rec2 - rec).max() < 1e-13


def test_thm2_reduced_bep(cfg1_proj):
    # Thm 2: a density satisfying the reduced BEP on γ_in satisfies the full BEP on γ.
    cfg, g, ps, P = cfg1_proj
    gidx = ps.list("gamma")
    ipos = np.searchsorted(gidx, ps.list("gamma_in"))
    epos = np.searchsorted(gidx, ps.list("gamma_ex"))
    rhs_full = uniform_values(12, len(gidx))
    A = np.eye(len(P)) - P
    # make the RHS a valid trace of a particular solution: project onto range(I - P)
    rhs = A @ rhs_full
    v = np.linalg.lstsq(A[ipos], rhs[ipos], rcond=None)[0]
    assert np.abs(A[ipos] @ v - rhs[ipos]).max() < 1e-11
    assert np.abs(A[epos] @ v - rhs[epos]).max() < 1e-11


def test_lsq_consistent_and_orthogonal():
    out = dpm.cfg1_outputs(get_config("cfg1"))
    B = out["B"]
    Cstar = uniform_values(13, B.shape[1])
    kappa = np.linalg.cond(B)
    assert abs(kappa - 48.7) < 0.5          # SURVEY probe P5: κ(B) = 48.7 at cfg1 (Cauchy basis)
    C = dpm.lstsq(B, B @ Cstar)
    assert np.abs(C - Cstar).max() < 1e-13 * kappa
    C2 = dpm.householder_lstsq(B, B @ Cstar)
    assert np.abs(C2 - Cstar).max() < 1e-13 * kappa
    # rhs ⟂ range(B) -> C = 0
    Q, _ = np.linalg.qr(B, mode="complete")
    r = Q[:, B.shape[1]:] @ uniform_values(14, B.shape[0] - B.shape[1])
    assert np.abs(dpm.lstsq(B, r)).max() < 1e-12
    # both LSQ algorithms agree on the real cfg1 right-hand side
    assert np.abs(dpm.householder_lstsq(B, out["rhs"]) - out["C"]).max() < 1e-13 * np.abs(out["C"]).max() * kappa


def manufactured_error(n):
    """SURVEY probe P6: zero-Neumann u* on the unit sphere, (I/dt - Δ)u = f, dt = 1e-2, L = 4."""
    from dpm_inputs.configs import Config
    cfg = Config("mms", n, -1.1, 1.1, "sphere", (0, 0, 0), (1, 1, 1), 4, "neumann0", 1e-2)
    g, ps = grid.point_sets_for(cfg)
    dt = cfg.dt
    x = g.coords()
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    R = np.sqrt(X ** 2 + Y ** 2 + Z ** 2)
    ustar = np.cos(np.pi * R) + Z * (1 - R ** 2 / 3) + (X ** 2 - Y ** 2) * (1 - R ** 2 / 2)
    lap = (-np.pi ** 2 * np.cos(np.pi * R) - 2 * np.pi * np.sin(np.pi * R) / R
           - 10.0 * Z / 3.0 - 7.0 * (X ** 2 - Y ** 2))
    f_paper = dt * (ustar / dt - lap)                      # L u* = (I - dt Δ) u*
    E, d, unit, foot = dpm.extension_matrix(g, ps, cfg.kind, cfg.center, cfg.semi, cfg.lmax, cfg.basis)
    _, B, _ = dpm.projection_and_bep(E, g, ps, dt)
    up = ap.solve(dpm.particular_rhs(f_paper, ps, dt), g.h, dt)
    C = dpm.lstsq(B, up.reshape(-1)[ps.list("gamma_in")])
    u = dpm.green(E @ C, f_paper, g, ps, dt)
    return np.abs(u - ustar)[ps.mplus].max()


@pytest.mark.slow
def test_manufactured_second_order():
    # Conjectured O(h^2 + dt); SURVEY probe P6 measured 9.41e-4 (N=32), 2.44e-4 (N=64)
    e32, e64 = manufactured_error(32), manufactured_error(64)
    assert abs(e32 / 9.41e-4 - 1) < 0.02 and abs(e64 / 2.44e-4 - 1) < 0.02
    assert np.log2(e32 / e64) > 1.9
