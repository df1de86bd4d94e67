"""R6 exact classification on the GPU: meshes with nodes exactly on Γ (sphere) or on the octant's
coordinate planes, where an fp64 test alone splits the ties; the point sets must equal the oracle's
exact-rational sets bit for bit, with every tie in M-."""
import numpy as np
import pytest
import torch

from oracle import dd as odd
from oracle import grid

pytestmark = pytest.mark.gpu

SETS = ["mplus", "gamma", "gamma_in", "gamma_ex", "band", "nplus"]


@pytest.fixture(scope="module")
def api():
    from paper_1811_03557_b200 import api as A
    assert torch.cuda.is_available()
    return A


@pytest.mark.parametrize("n", [65, 109, 131])
def test_sphere_ties_bit_exact(api, n):
    # unit sphere in [-1.1, 1.1]^3: 150 nodes exactly on Γ at each of these n (tests/test_oracle_grid.py)
    c = api.DPM(n, -1.1, 1.1, "sphere", (0, 0, 0), (1, 1, 1), 2, 1e-3, "cauchy")
    g = grid.Grid(n, -1.1, 1.1)
    ps = grid.point_sets(g, "sphere", (0.0, 0.0, 0.0), (1.0, 1.0, 1.0))
    for w in SETS:
        assert np.array_equal(c.copy_set(w), ps.list(w)), (n, w)
    assert c.info["n_exact_ties"] >= 150 and c.info["n_exact_ties_inside"] < c.info["n_exact_ties"]


def test_ellipsoid_and_offcentre_sphere_bit_exact(api):
    # decimal constants with several digits (R6 reads them as decimals): an off-centre sphere and an
    # ellipsoid whose semi-axes make ties likely on a fine mesh
    for kind, center, semi, n, lo, hi in (("sphere", (0.125, -0.125, 0.0), (0.75, 0.75, 0.75), 63, -1.0, 1.0),
                                          ("ellipsoid", (0.0, 0.0, 0.0), (0.9, 0.6, 0.5), 89, -1.0, 1.0)):
        c = api.DPM(n, lo, hi, kind, center, semi, 2, 1e-3, "cauchy")
        ps = grid.point_sets(grid.Grid(n, lo, hi), kind, center, semi)
        for w in SETS:
            assert np.array_equal(c.copy_set(w), ps.list(w)), (kind, w)


@pytest.mark.parametrize("n", [23, 35])
def test_octant_plane_ties_bit_exact(api, n):
    # box [-0.1, 1.1]^3: node i = (n+1)/12 - 1 lies exactly on each coordinate plane (R24: -> M-)
    o = odd.setup(n, 2, 2).octants[0]
    g = api.Octant(n, -0.1, 1.1, 0, 1.0, 2, 2, 1e-3)
    for w in SETS:
        assert np.array_equal(g.copy_set(w), o.ps.list(w)), (n, w)
    assert g.info["n_exact_ties"] > 0
