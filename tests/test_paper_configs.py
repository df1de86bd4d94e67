"""The paper-test inputs (dpm_inputs.test_a_config / test_b_config) against the paper's stated parameters."""
import math

from dpm_inputs import paper_mesh
from dpm_inputs import test_a_config as make_test_a   # (aliases: not collected as tests)
from dpm_inputs import test_b_config as make_test_b


def test_test_a_config_matches_paper():
    # Test A: ρ0 = 1000 exp(-100 |x|^2), c0 = 500 exp(-50 |x|^2); sphere r = 0.5 at the origin
    # (P:596); one zonal harmonic per term of the 3-term extension; dt = 1e-8 to T = 1e-6 (Tables 1-3)
    for N in (36, 68, 132, 260, 516):
        cfg = make_test_a(N)
        assert cfg.kind == "sphere" and cfg.center == (0.0, 0.0, 0.0) and cfg.semi == (0.5, 0.5, 0.5)
        assert cfg.ic_center == (0.0, 0.0, 0.0) and cfg.ic_rho == (1000.0, 100.0) and cfg.ic_c == (500.0, 50.0)
        assert cfg.basis == "neumann0_zonal" and cfg.lmax == 0 and cfg.K == 2
        assert cfg.dt == 1e-8 and cfg.steps == 100 and abs(cfg.steps * cfg.dt - 1e-6) < 1e-20
        n, lo, hi, h = paper_mesh(N, 0.5)
        assert (cfg.n, cfg.lo, cfg.hi) == (n, lo, hi) and math.isclose(h, 1.0 / (N - 4), rel_tol=1e-15)


def test_test_b_config_matches_paper():
    # Test B: ρ0 = 2000 exp(-100 (x^2 + y^2 + (z - 0.25)^2)), c0 = 0; 2-term extension with
    # zonal harmonics on Γ; dt = 0.5 h^2 before blow-up
    for N, H in ((127, 150), (255, 300)):
        cfg = make_test_b(N, H)
        assert cfg.ic_center == (0.0, 0.0, 0.25) and cfg.ic_rho == (2000.0, 100.0) and cfg.ic_c[0] == 0.0
        assert cfg.basis == "neumann0_2term_zonal" and cfg.lmax + 1 == H and cfg.K == H
        h = 1.0 / (N - 4)
        assert math.isclose(cfg.dt, 0.5 * h * h, rel_tol=1e-14)
        assert cfg.semi == (0.5, 0.5, 0.5)
