"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no point sets, no transforms, no
stencils): only the five BASELINE.json configurations as plain parameters and
seeded random-number draws.  Both the oracle (``oracle/``) and the CUDA path
(``paper_1811_03557_b200``) consume what it returns; neither imports the other.

Configurations (BASELINE.json ``configs``; readings R1-R31 of SURVEY.md §8(c)):

* cfg1 - single DPM auxiliary batch, unit sphere in [-1.1,1.1]^3, N=16, dt=1e-3,
  L=4 Cauchy basis {Y, d*Y} (K=50) + 1 particular RHS of U(-1,1) from seed 0 (R22).
* cfg2 - PKS, unit sphere in [-1.1,1.1]^3, N=32, dt cap 1e-4, L=6, zero-Neumann
  basis {Y, d^2/2*Y}, 10 steps.
* cfg3 - PKS, ellipsoid (0.9,0.6,0.5) in [-1,1]^3, N=64, dt cap 2e-5, L=10,
  ICs centred at (0.2,0,0), 100 steps.
* cfg4 - throughput: N=128, [-1.1,1.1]^3, dt=1e-5, 578 RHS of U(-1,1) on the
  spherical shell band of r=1 (R21).
* cfg5 - 8-octant DD (R24), N=128 per octant (not built in round 1).
"""
from .configs import CONFIGS, Config, get_config, paper_mesh, test_a_config, test_b_config  # noqa: F401
from .rng import uniform_values, cfg1_particular_values, cfg4_band_values  # noqa: F401
