"""Pins for oracle/pks.py: the FV/IMEX scheme, CFL, Steps 3-7."""
import math

import numpy as np
import pytest

from dpm_inputs import get_config
from dpm_inputs.rng import uniform_values
from oracle import grid, pks


def test_minmod_examples():
    # SPEC S:197-199
    assert pks.minmod(2.0, 1.5, 1.0) == 1.0
    assert pks.minmod(-2.0, 1.0, 3.0) == 0.0
    assert pks.minmod(-1.0, -2.0, -3.0) == -1.0


@pytest.fixture(scope="module")
def cfg2_sets():
    return grid.point_sets_for(get_config("cfg2"))


def test_slopes_linear_and_spike(cfg2_sets):
    g, ps = cfg2_sets
    n, h = g.n, g.h
    x = g.coords()
    X = np.broadcast_to(x[:, None, None], (n, n, n))
    R = np.zeros((n + 2,) * 3)
    R[1:-1, 1:-1, 1:-1] = np.where(ps.nplus, X, 0.0)
    S = pks.limited_slopes(R, ps.nplus_lat, h)
    mp = np.zeros_like(ps.nplus_lat)
    mp[1:-1, 1:-1, 1:-1] = ps.mplus
    interior = mp & np.roll(mp, 1, 0) & np.roll(mp, -1, 0)
    assert np.allclose(S[0][interior], 1.0, rtol=1e-12)       # linear exactness
    assert np.all(S[1][interior] == 0) and np.all(S[2][interior] == 0)
    # spike -> slope 0 at the spike
    R2 = np.zeros_like(R)
    c = n // 2 + 1
    R2[c, c, c] = 1.0
    S2 = pks.limited_slopes(R2, ps.nplus_lat, h)
    assert all(s[c, c, c] == 0 for s in S2)


def test_convection_quadratic_exact(cfg2_sets):
    # ρ̄ ≡ ρ0, c = x^2 -> g = 2 χ ρ0 on every M+ cell
    g, ps = cfg2_sets
    n = g.n
    x = g.coords()
    c = np.where(ps.nplus, np.broadcast_to(x[:, None, None] ** 2, (n, n, n)), 0.0)
    rho = np.where(ps.nplus, 3.0, 0.0)
    gconv = pks.convection(rho, c, ps, g.h, 1.0)
    assert np.abs(gconv[ps.mplus] - 6.0).max() < 1e-9
    # c constant -> g ≡ 0 exactly
    assert np.all(pks.convection(rho, np.where(ps.nplus, 5.0, 0.0), ps, g.h, 1.0) == 0.0)


def test_assemble_rhs_and_cfl(cfg2_sets):
    # SPEC S:224-226 and S:233-235
    fr, fc = pks.assemble_rhs(np.array(2.0), np.array(4.0), np.array(1.0), 0.5)
    assert fr == 1.5 and fc == 3.0
    g, ps = cfg2_sets
    n = g.n
    x = g.coords()
    c = np.where(ps.nplus, np.broadcast_to(5.0 * x[:, None, None], (n, n, n)), 0.0)
    assert abs(pks.cfl_dt(c, ps, g.h, 1.0) - g.h / 30.0) < 1e-15
    assert pks.cfl_dt(np.where(ps.nplus, 1.0, 0.0), ps, g.h, 1.0) == np.inf


def test_conservation_identity_and_positivity(cfg2_sets):
    # ρ̄ = mean of the six one-sided face values; Thm 3 flux split: f_ρ >= 0 under CFL
    g, ps = cfg2_sets
    n, h = g.n, g.h
    rho = np.where(ps.nplus, np.abs(uniform_values(21, (n, n, n))), 0.0)
    c = np.where(ps.nplus, np.abs(uniform_values(22, (n, n, n))), 0.0)
    R = np.zeros((n + 2,) * 3)
    R[1:-1, 1:-1, 1:-1] = rho
    S = pks.limited_slopes(R, ps.nplus_lat, h)
    faces = sum((R + 0.5 * h * s) + (R - 0.5 * h * s) for s in S) / 6.0
    assert np.abs(faces - R).max() < 1e-15
    for s in S:   # limited reconstruction is non-negative
        assert (R + 0.5 * h * s).min() >= -1e-15 and (R - 0.5 * h * s).min() >= -1e-15
    dt = pks.cfl_dt(c, ps, h, 1.0)
    fr, _ = pks.assemble_rhs(rho, c, pks.convection(rho, c, ps, h, 1.0), dt)
    assert fr[ps.mplus].min() >= -1e-12


@pytest.mark.slow
def test_cfg2_run_survey_probe_values():
    # SURVEY probe P11 (independent probe of readings R13-R20, cfg2, 10 steps):
    # dt = 4.6352e-6 every step, 1 BEP build, max ρ 2.125875e3, mass drift -4.3e-15.
    o = pks.PKSOracle(get_config("cfg2"))
    rho0, c0 = o.initial_state()
    m0 = o.mass(rho0)
    rho, c, logs = o.run()
    assert o.builds == 1
    assert all(abs(l["dt"] / 4.6352e-6 - 1) < 1e-4 for l in logs)
    assert abs(rho.max() / 2.125875e3 - 1) < 1e-6
    assert abs(logs[-1]["mass"] - m0) < 1e-12 * m0
    assert abs(m0 / 5.5683279893 - 1) < 1e-9
    # positivity (Thm 3) up to round-off
    assert rho.min() > -1e-9 * rho.max() and c.min() > -1e-9 * c.max()


# ------------------------------------------------------------------ diagnostics
def _diag_loops(rho, c, g, ps, center):
    """Brute force over the nodes with explicit neighbour lookups (independent of the padded-array form)."""
    n, h = g.n, g.h
    x = g.coords()
    mass = second = free = 0.0
    cv = lambda i, j, k: c[i, j, k] if 0 <= i < n and 0 <= j < n and 0 <= k < n else 0.0   # noqa: E731
    for i in range(n):
        for j in range(n):
            for k in range(n):
                if not ps.mplus[i, j, k]:
                    continue
                r, cc = rho[i, j, k], c[i, j, k]
                mass += r
                second += ((x[i] - center[0]) ** 2 + (x[j] - center[1]) ** 2 + (x[k] - center[2]) ** 2) * r
                g2 = ((cv(i + 1, j, k) - cv(i - 1, j, k)) ** 2 + (cv(i, j + 1, k) - cv(i, j - 1, k)) ** 2
                      + (cv(i, j, k + 1) - cv(i, j, k - 1)) ** 2)
                free += (r * math.log(r) if r > 0 else 0.0) - r * cc + 0.5 * cc * cc + g2 / (8 * h * h)
    return {"mass": h ** 3 * mass, "second_moment": h ** 3 * second, "free_energy": h ** 3 * free}


def test_diagnostics_brute_force_and_closed_forms():
    cfg = get_config("cfg1")
    g, ps = grid.point_sets_for(cfg)
    rng = np.random.default_rng(3)
    rho = rng.uniform(-0.1, 2.0, size=(g.n,) * 3)     # includes ρ <= 0 (ρ ln ρ := 0, R35)
    c = rng.uniform(0.0, 3.0, size=(g.n,) * 3)
    d = pks.diagnostics(rho, c, g, ps, cfg.center)
    b = _diag_loops(rho, c, g, ps, cfg.center)
    for k in d:
        assert abs(d[k] - b[k]) <= 1e-12 * abs(b[k]), k
    # constant state on cfg2 (no M+ node next to the ghost layer there, unlike cfg1's 72, R5):
    # no gradient term, E = h^3 |M+| (ρ ln ρ - ρ c + c^2/2)
    cfg = get_config("cfg2")
    g, ps = grid.point_sets_for(cfg)
    assert ps.ghosts_in_nplus == 0
    nm = int(ps.mplus.sum())
    d = pks.diagnostics(np.full((g.n,) * 3, 2.0), np.full((g.n,) * 3, 3.0), g, ps, cfg.center)
    assert abs(d["free_energy"] - g.h ** 3 * nm * (2 * math.log(2) - 6 + 4.5)) < 1e-13 * nm * g.h ** 3
    assert abs(d["mass"] - 2 * g.h ** 3 * nm) < 1e-12
    # linear c = a x: the central difference is exact, gradient term h^3 |M+| a^2 / 2
    a = 1.7
    X = np.broadcast_to(g.coords()[:, None, None], (g.n,) * 3)
    d = pks.diagnostics(np.zeros((g.n,) * 3), a * X, g, ps, cfg.center)
    ref = g.h ** 3 * (0.5 * a * a * np.sum(X[ps.mplus] ** 2) + nm * a * a / 2)
    assert abs(d["free_energy"] - ref) < 1e-12 * ref


def test_second_moment_continuum_limit():
    # ρ = 1 on M+ of the unit ball: M_h -> ∫_B |x|^2 dx = 4π/5 (first order in h: staircase boundary)
    cfg = get_config("cfg2")
    g, ps = grid.point_sets_for(cfg)
    d = pks.diagnostics(np.ones((g.n,) * 3), np.zeros((g.n,) * 3), g, ps, cfg.center)
    assert abs(d["second_moment"] / (4 * math.pi / 5) - 1) < 0.1
    assert abs(d["mass"] / (4 * math.pi / 3) - 1) < 0.1


def test_cell_average_initial_state():
    # R36: ρ̄0 on M+ \ γ is the cell average of ρ0 = A exp(-a |x - x0|^2); against tensor-product
    # Gauss-Legendre quadrature over the cell (exact to ~1e-15 for these smooth integrands)
    cfg = get_config("cfg3")   # off-centre IC (0.2, 0, 0) on the ellipsoid
    o = pks.PKSOracle(cfg)
    rho_pt, _ = o.initial_state()
    rho, c = o.initial_state(rho_cell_average=True)
    g, ps = o.g, o.ps
    x = g.coords()
    t, w = np.polynomial.legendre.leggauss(16)
    A, a = cfg.ic_rho
    x0 = np.asarray(cfg.ic_center)
    inner = ps.mplus & ~ps.gamma
    idx = np.argwhere(inner)
    rng = np.random.default_rng(0)
    for i, j, k in idx[rng.choice(len(idx), 25, replace=False)]:
        pts = [x[q] + 0.5 * g.h * t for q in (i, j, k)]
        f = [np.sum(0.5 * w * np.exp(-a * (pts[d] - x0[d]) ** 2)) for d in range(3)]
        ref = A * f[0] * f[1] * f[2]
        assert abs(rho[i, j, k] - ref) <= 1e-13 * A, (i, j, k)
    # γ keeps the foot-point values (R14) and c stays a point value
    assert np.array_equal(rho[ps.gamma], rho_pt[ps.gamma])
    assert np.array_equal(c, o.initial_state()[1])
    # averaging a peaked Gaussian lowers the maximum
    assert rho[inner].max() < rho_pt[inner].max()


def test_sequential_coupling_variant():
    # coupling = 1 changes only the c equation's ρ̄ (ρ̄^{i+1} instead of ρ̄^i): after one step ρ is
    # identical and c differs by dt (ρ̄^{i+1} - ρ̄^i) through the c solve
    cfg = get_config("cfg2")
    a, b = pks.PKSOracle(cfg, dt_rule=1), pks.PKSOracle(cfg, dt_rule=1, coupling=1)
    r0, c0 = a.initial_state()
    ra, ca, _ = a.step(r0, c0)
    rb, cb, _ = b.step(r0, c0)
    assert np.array_equal(ra, rb)
    assert 0 < np.abs(ca - cb).max() < 1e-2 * np.abs(ca).max()
    # the c equation does not involve g, so the sequential c^{i+1} is exactly the printed
    # scheme's c output from the state (ρ̄^{i+1}, c^i) at the same dt
    _, c_seq, _ = pks.PKSOracle(cfg, dt_rule=1).step(ra, c0)
    assert np.abs(cb - c_seq).max() <= 1e-13 * np.abs(cb).max()


@pytest.mark.parametrize("s", [2.0, -3.0])
def test_upwind_direction_hand_computed(cfg2_sets, s):
    # the face value of ρ is the LEFT reconstruction ρ_j + h/2 σ_j where ∇c > 0 and the RIGHT
    # one ρ_{j+1} - h/2 σ_{j+1} otherwise.  ρ̄ = e^{kx} (non-constant and not linear, so the two sides
    # differ), c = s x (∇c = s on every x face, 0 on the y and z faces).  Where the x stencil j-2..j+2
    # lies in N+, minmod picks the central slope σ_j = e^{k x_j} sinh(kh)/h (kh = 0.3), so by hand
    #   s > 0:  g_j = χ s (1 + sinh(kh)/2)(e^{k x_j} - e^{k x_{j-1}}) / h,
    #   s < 0:  g_j = χ s (1 - sinh(kh)/2)(e^{k x_{j+1}} - e^{k x_j}) / h.
    # Swapping the upwind direction changes g by ~2e-3 relative, far above the 1e-12 tolerance.
    g, ps = cfg2_sets
    n, h = g.n, g.h
    k = 0.3 / h
    chi = 1.7
    x = g.coords()
    X = np.broadcast_to(x[:, None, None], (n, n, n))
    rho = np.where(ps.nplus, np.exp(k * X), 0.0)
    c = np.where(ps.nplus, s * X, 0.0)
    gconv = pks.convection(rho, c, ps, h, chi)
    npl = ps.nplus_lat
    ok = np.ones((n, n, n), dtype=bool)
    for d in (-2, -1, 0, 1, 2):
        ok &= np.roll(npl, -d, axis=0)[1:-1, 1:-1, 1:-1]   # node i + d along x in N+
    ok &= ps.mplus
    ok[:2] = False                                          # no wrap-around of np.roll
    ok[-2:] = False
    # the y / z neighbours of a checked cell must be in N+ too (their faces carry ∇c = 0 -> no flux,
    # but c must be the same linear function there)
    for ax in (1, 2):
        for d in (-1, 1):
            ok &= np.roll(npl, -d, axis=ax)[1:-1, 1:-1, 1:-1]
    e = np.exp(k * X)
    em, ep = np.exp(k * (X - h)), np.exp(k * (X + h))
    sh = np.sinh(k * h)
    if s > 0:
        want = chi * s * (1 + sh / 2) * (e - em) / h
    else:
        want = chi * s * (1 - sh / 2) * (ep - e) / h
    assert ok.sum() > 1000
    assert np.abs(gconv[ok] - want[ok]).max() <= 1e-12 * np.abs(want[ok]).max()
    wrong = chi * s * ((1 - sh / 2) * (ep - e) if s > 0 else (1 + sh / 2) * (e - em)) / h
    assert np.abs(wrong[ok] - want[ok]).max() > 1e-4 * np.abs(want[ok]).max()
