"""The BASELINE.json configurations as plain parameter records (no method arithmetic).

Grid convention: the box faces [lo, hi]^3 are the Dirichlet
(ghost) nodes; ``n`` is the number of unknowns per axis; h = (hi-lo)/(n+1).
"""
from dataclasses import dataclass, field
from typing import Optional, Tuple


@dataclass(frozen=True)
class Config:
    name: str
    n: int                       # unknowns per axis (R2)
    lo: float                    # box = [lo, hi]^3 (R1, R3)
    hi: float
    kind: str                    # "sphere" | "ellipsoid"
    center: Tuple[float, float, float]
    semi: Tuple[float, float, float]   # sphere: (r, r, r)
    lmax: int                    # spherical-harmonic degree L
    basis: str                   # "cauchy" {Y, d*Y} | "neumann0" {Y, d^2/2*Y}  (R9); "*_zonal": P_l^0 only
    dt: float                    # AP dt (cfg1, cfg4) or the PKS dt cap (cfg2, cfg3, cfg5)
    steps: int = 0               # PKS steps (0 = not a PKS config)
    batch: int = 0               # number of RHS in the throughput config
    # PKS initial conditions rho0 = A_rho exp(-a_rho |x - ic_center|^2), c0 = A_c exp(-a_c |x - ic_center|^2)
    ic_center: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    ic_rho: Tuple[float, float] = (1000.0, 100.0)
    ic_c: Tuple[float, float] = (500.0, 50.0)
    chi: float = 1.0             # R27: alpha = gamma_rho = gamma_c = chi = 1
    deg_if: int = 0              # cfg5: interface polynomial degree (R24); lmax is the cap SH degree

    @property
    def K(self) -> int:
        nb = self.lmax + 1 if self.basis.endswith("_zonal") else (self.lmax + 1) ** 2
        return nb if self.basis.startswith("neumann0_2term") else 2 * nb


CONFIGS = {
    "cfg1": Config("cfg1", 16, -1.1, 1.1, "sphere", (0.0, 0.0, 0.0), (1.0, 1.0, 1.0), 4, "cauchy", 1e-3,
                   batch=51),
    "cfg2": Config("cfg2", 32, -1.1, 1.1, "sphere", (0.0, 0.0, 0.0), (1.0, 1.0, 1.0), 6, "neumann0", 1e-4,
                   steps=10),
    "cfg3": Config("cfg3", 64, -1.0, 1.0, "ellipsoid", (0.0, 0.0, 0.0), (0.9, 0.6, 0.5), 10, "neumann0", 2e-5,
                   steps=100, ic_center=(0.2, 0.0, 0.0)),
    "cfg4": Config("cfg4", 128, -1.1, 1.1, "sphere", (0.0, 0.0, 0.0), (1.0, 1.0, 1.0), 16, "cauchy", 1e-5,
                   batch=578),
    # cfg5 (R24, R3): 8 octant subdomains, each on its own canonical box [-0.1, 1.1]^3 with
    # n = 128; cap SH degree 12 and interface degree 12 (K = 884); dt cap 1e-5; 50 steps.
    "cfg5": Config("cfg5", 128, -0.1, 1.1, "octant8", (0.0, 0.0, 0.0), (1.0, 1.0, 1.0), 12, "neumann0", 1e-5,
                   steps=50, deg_if=12),
}


def get_config(name: str) -> Config:
    return CONFIGS[name]


def paper_mesh(N: int, r: float):
    """The paper's single-domain mesh: N cells per axis on [-r-2h, r+2h]^3, h = 2r/(N-4),
    cell centres at -r-2h + (j-1/2)h.  In this repo's convention (R1: box faces = ghost nodes,
    n unknowns, node i at lo + (i+1)h) that is n = N, lo = -r - 5h/2, hi = r + 5h/2."""
    h = 2.0 * r / (N - 4)
    return N, -r - 2.5 * h, r + 2.5 * h, h


def test_a_config(N: int, dt: float = 1e-8, steps: int = 100) -> Config:
    """The paper's Test A for the convergence study, single domain: sphere
    r = 0.5, rho0 = 1000 exp(-100 r^2), c0 = 500 exp(-50 r^2); the 3-term extension (beta = 1) with
    one zonal harmonic per term; fixed dt = 1e-8 to T = 1e-6 (Tables 1-3)."""
    n, lo, hi, h = paper_mesh(N, 0.5)
    return Config(f"testA{N}", n, lo, hi, "sphere", (0.0, 0.0, 0.0), (0.5, 0.5, 0.5), 0, "neumann0_zonal", dt,
                  steps=steps, ic_rho=(1000.0, 100.0), ic_c=(500.0, 50.0))


def test_b_config(N: int = 127, harmonics: int = 150) -> Config:
    """The paper's Test B, single domain: sphere r = 0.5 at the origin,
    rho0 = 2000 exp(-100 (x^2 + y^2 + (z - 0.25)^2)), c0 = 0; the 2-term extension with zero
    Neumann data (beta = 0) and `harmonics` zonal modes; dt = 0.5 h^2 before blow-up
    and the CFL rule after."""
    n, lo, hi, h = paper_mesh(N, 0.5)
    return Config(f"testB{N}", n, lo, hi, "sphere", (0.0, 0.0, 0.0), (0.5, 0.5, 0.5), harmonics - 1,
                  "neumann0_2term_zonal", 0.5 * h * h, ic_center=(0.0, 0.0, 0.25), ic_rho=(2000.0, 100.0),
                  ic_c=(0.0, 1.0))
