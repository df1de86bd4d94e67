"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct fp64 NumPy implementation of what the DPM hot
path computes, written from the paper (/root/reference/PAPER.md, cited as P:<line>)
and the readings R1-R31 of SURVEY.md §8(c) (listed again in DESIGN.md).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA path (``paper_1811_03557_b200``) and never imports it.

Modules
-------
grid      grid (R1) + exact rational classification (R6) + point sets of Def. 1
ap        auxiliary-problem solve by direct-summation DST-I (R4, R26) + dense LU
geometry  foot points, signed distance, SH angles on sphere / ellipsoid (R10)
sh        real orthonormal spherical harmonics without Condon-Shortley phase (R8)
dpm       extension matrix, difference potentials, P_gamma, reduced BEP, LSQ, Green
pks       minmod/upwind flux, IMEX right-hand sides, CFL, the time step

Parity pins: every function is pinned in tests/test_oracle_*.py against closed forms,
brute force, invariants or the paper's theorems; see DESIGN.md "Oracle pins".
"""
