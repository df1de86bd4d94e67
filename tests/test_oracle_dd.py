"""Pins of the octant-DD oracle (oracle/dd.py).  The paper has no octant DD
(parity unpinned vs the paper); the pins are the survey's independent probe counts, exact
extension identities, the single-octant DPM convergence and the 8-fold reflection symmetry."""
import numpy as np
import pytest

from oracle import dd, dpm, grid

N16 = 16


def test_cfg5_counts_and_piece_multiplicity():
    """SURVEY §8(a) cfg5 row (probe P1) and probe P9 at n = 128 per octant, box [-0.1, 1.1]^3."""
    g = grid.Grid(128, -0.1, 1.1)
    ps = grid.point_sets_from_mask(g, grid.octant_inside_mask(g))
    assert (int(ps.mplus.sum()), int(ps.gamma.sum()), int(ps.gamma_in.sum()), int(ps.gamma_ex.sum()),
            int(ps.band.sum())) == (657356, 84431, 41734, 42697, 86365)
    A = dd.piece_assignment(g, ps)
    mult = np.bincount(A.sum(axis=1), minlength=4)
    assert list(mult) == [0, 78877, 5478, 76]                     # every γ point covered (P9)
    gin = np.searchsorted(ps.list("gamma"), ps.list("gamma_in"))
    assert int(A[gin].sum()) == 44145                             # BEP rows incl. duplicates (P9)


def test_legendre_and_plane_basis():
    x = np.linspace(-1, 1, 7)
    P = dd.legendre(4, x)
    assert np.allclose(P[:, 2], 0.5 * (3 * x ** 2 - 1), atol=1e-15)
    assert np.allclose(P[:, 4], (35 * x ** 4 - 30 * x ** 2 + 3) / 8, atol=1e-15)
    modes = dd.plane_modes(3)
    assert len(modes) == 10 and modes[:4] == [(0, 0), (1, 0), (0, 1), (2, 0)]


def _ustar(X):
    x, y, z = X[..., 0], X[..., 1], X[..., 2]
    r = np.sqrt(x * x + y * y + z * z)
    return np.cos(np.pi * r) + z * (1 - r * r / 3) + (x * x - y * y) * (1 - r * r / 2)


def _lap(X):
    x, y, z = X[..., 0], X[..., 1], X[..., 2]
    r = np.sqrt(x * x + y * y + z * z)
    return -np.pi ** 2 * np.cos(np.pi * r) - 2 * np.pi / r * np.sin(np.pi * r) - 10 * z / 3 - 7 * (x * x - y * y)


def _grad(X):
    x, y, z = X[..., 0], X[..., 1], X[..., 2]
    r = np.sqrt(x * x + y * y + z * z)
    dc = -np.pi * np.sin(np.pi * r) / r
    return np.stack([dc * x - 2 * x * z / 3 + 2 * x * (1 - r * r / 2) - x * (x * x - y * y),
                     dc * y - 2 * y * z / 3 - 2 * y * (1 - r * r / 2) - y * (x * x - y * y),
                     dc * z + (1 - r * r / 3) - 2 * z * z / 3 - z * (x * x - y * y)], axis=-1)


def test_extension_rows_reproduce_exact_cauchy_data():
    """Each piece's extension row, fed the exact Cauchy data of a smooth u*, reproduces u* at the
    γ points up to the Taylor remainder of the piece (cap: 3-term with ∂_n u = 0, plane: 2-term):
    plane error <= d^2/2 max|∂²_a u*| (<= 12), in every octant (signs of the reflected frames)."""
    st = dd.setup(N16, 2, 2)
    for o in st.octants:
        P = dpm.gamma_points(o.g, o.ps) * o.sigma
        tru = _ustar(P)
        for a in range(3):
            F = P.copy()
            F[:, a] = 0.0
            ext = _ustar(F) + P[:, a] * _grad(F)[:, a]
            m = o.assign[:, 1 + a]
            assert np.all(np.abs(ext - tru)[m] <= 6.0 * P[m, a] ** 2 + 1e-14)
        r = np.linalg.norm(P, axis=1)
        f = P / r[:, None]
        d = r - 1.0
        ext = _ustar(f) + 0.5 * d * d * (np.pi ** 2 - 2 * f[:, 2] - 4 * (f[:, 0] ** 2 - f[:, 1] ** 2))
        m = o.assign[:, 0]
        assert np.abs(ext - tru)[m].max() <= 4.0 * o.g.h ** 3 * 10


@pytest.mark.slow
def test_octant_green_second_order_with_true_density():
    """The octant's potentials + Green's formula with the exact density reproduce u* on M+ at 2nd
    order (pins the octant grid, sets and AP solve geometry)."""
    dt, errs = 1e-2, []
    for n in (16, 32):
        st = dd.setup(n, 0, 0)
        o = st.octants[0]
        x = o.g.coords()
        X = np.stack(np.meshgrid(x, x, x, indexing="ij"), -1)
        f = dt * (_ustar(X) / dt - _lap(X))
        ug = _ustar(dpm.gamma_points(o.g, o.ps))
        u = dpm.green(ug, f, o.g, o.ps, dt)
        errs.append(np.abs(u - _ustar(X))[o.ps.mplus].max())
    assert errs[1] < errs[0] / 3.0, errs


def test_reflection_symmetry_of_coupled_pks():
    """An origin-centred IC is invariant under the 8 reflections, so every octant's canonical-frame
    fields must coincide after coupled steps (fails on any sign error in the shared bases)."""
    o = dd.DDPKSOracle(12, 2, 2, 1e-3, 2)
    state, logs = o.run()
    ref = state[0]
    for rho, c in state[1:]:
        assert np.abs(rho - ref[0]).max() <= 1e-10 * np.abs(ref[0]).max()
        assert np.abs(c - ref[1]).max() <= 1e-10 * np.abs(ref[1]).max()
    assert logs[0]["rebuilt"] and o.builds >= 1


def test_column_signs_match_the_octant_extensions():
    # E_s = E_0 diag(S_s) for every octant (the reflection parity of the cap SH and plane Legendre bases)
    st = dd.setup(16, 4, 4)
    S = dd.column_signs(st)
    E0 = st.octants[0].Eraw
    for s, o in enumerate(st.octants):
        assert np.abs(o.Eraw - E0 * S[s]).max() <= 1e-13 * np.abs(E0).max()
        assert np.abs(o.A - st.octants[0].A * S[s]).max() <= 1e-13 * np.abs(E0).max()
    assert set(np.unique(S)) == {-1.0, 1.0}


def test_symmetric_reduction_equals_the_stacked_oracle():
    # the one-octant symmetric oracle (used for cfg5 at its configured size) against the full 8-octant
    # stacked oracle on the same symmetric IC: same dt sequence, same fields in every octant
    steps, cap = 3, 1e-3
    full = dd.DDPKSOracle(16, 4, 4, cap, steps)
    sym = dd.DDPKSOracleSymmetric(16, 4, 4, cap, steps)
    sf, lf = full.run()
    ss, ls = sym.run()
    for (ro, co) in sf:
        assert np.abs(ro - ss[0]).max() <= 1e-12 * np.abs(ro).max()
        assert np.abs(co - ss[1]).max() <= 1e-12 * np.abs(co).max()
    for a, b in zip(lf, ls):
        assert a["dt"] == b["dt"] and a["rebuilt"] == b["rebuilt"]
        assert abs(a["mass"] - b["mass"]) <= 1e-12 * abs(a["mass"])
