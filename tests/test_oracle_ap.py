"""Pins for oracle/ap.py: the AP solved by direct-summation DST-I."""
import itertools

import numpy as np
import pytest

from dpm_inputs.rng import random_boxes
from oracle import ap


def test_eigenvalue_closed_form():
    # N=4, h=1 -> λ_1 = 2(1 - cos(pi/5)) ≈ 0.381966
    lam = ap.eigenvalues(4, 1.0)
    assert abs(lam[0] - 2 * (1 - np.cos(np.pi / 5))) < 1e-15
    assert abs(lam[0] - 0.3819660112501051) < 1e-15
    # scaling with h: h = 0.5 -> 4x
    assert np.allclose(ap.eigenvalues(4, 0.5), 4 * lam, rtol=1e-15)


@pytest.mark.parametrize("n", [4, 7, 16, 33])
def test_sine_matrix_square(n):
    # textbook: S^2 = ((n+1)/2) I
    S = ap.sine_matrix(n)
    assert np.abs(S @ S - (n + 1) / 2 * np.eye(n)).max() < 1e-12 * n


@pytest.mark.parametrize("n", [5, 8])
def test_eigenfunction(n):
    # q = (1/dt + λa + λb + λc) S_abc  ->  u = S_abc
    h, dt = 0.3, 0.01
    lam = ap.eigenvalues(n, h)
    j = np.arange(1, n + 1)
    for a, b, c in [(1, 1, 1), (2, n, 3), (n, n - 1, 1)]:
        Sabc = np.einsum("i,j,k->ijk", np.sin(np.pi * a * j / (n + 1)), np.sin(np.pi * b * j / (n + 1)),
                         np.sin(np.pi * c * j / (n + 1)))
        q = (1 / dt + lam[a - 1] + lam[b - 1] + lam[c - 1]) * Sabc
        assert np.abs(ap.solve(q, h, dt) - Sabc).max() < 1e-13


@pytest.mark.parametrize("n", [4, 6, 8])
def test_dense_lu(n):
    q = random_boxes(1, 1, n)[0]
    h, dt = 2.2 / (n + 1), 1e-3
    u = ap.solve(q, h, dt)
    ud = ap.dense_solve(q, h, dt)
    assert np.abs(u - ud).max() / np.abs(ud).max() < 1e-13


@pytest.mark.parametrize("n,dt", [(16, 1e-3), (32, 1e-5), (31, 0.5)])
def test_residual(n, dt):
    # ||(I/dt - Δ_h)u - q||_inf <= 1e-11 (1 + ||q||_inf)  (scaled form)
    q = random_boxes(2, 2, n)
    h = 2.2 / (n + 1)
    u = ap.solve(q, h, dt)
    r = ap.apply_operator(u, h, dt) - q
    assert np.abs(r).max() <= 1e-11 * (1 + np.abs(q).max())


def test_symmetry_and_max_principle():
    n = 9
    q = np.zeros((n, n, n))
    q[4, 4, 4] = 1.0
    u = ap.solve(q, 0.2, 0.05)
    for perm in itertools.permutations(range(3)):
        v = np.transpose(u, perm)
        for flips in itertools.product([False, True], repeat=3):
            w = v
            for ax, f in enumerate(flips):
                if f:
                    w = np.flip(w, axis=ax)
            assert np.abs(w - u).max() < 1e-15 * np.abs(u).max() * 10
    # M-matrix: q >= 0 => u >= 0
    qp = np.abs(random_boxes(3, 1, n)[0])
    assert ap.solve(qp, 0.2, 0.05).min() >= -1e-12 * qp.max()


def test_linearity():
    n = 12
    q1, q2 = random_boxes(4, 2, n)
    h, dt = 0.1, 1e-2
    lhs = ap.solve(2.5 * q1 - 0.5 * q2, h, dt)
    rhs = 2.5 * ap.solve(q1, h, dt) - 0.5 * ap.solve(q2, h, dt)
    assert np.abs(lhs - rhs).max() < 1e-12 * np.abs(rhs).max()
