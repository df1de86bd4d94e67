"""Auxiliary-problem (AP) solver — oracle (test infrastructure only).

The discrete AP (`eqn:discrete_ap`, `eqn:discrete_ap_boundary`):
    L v = q on M0,   v = 0 on N0 \\ M0,
with L the 7-point operator.  The paper writes L = I - dt Δ_h; the ABI
solves the equivalent scaled form (I/dt - Δ_h) u = q: identical u
when q_ABI = q_paper / dt.

Plain definition used here: the 3D type-I discrete sine transform diagonalises the
Dirichlet 7-point Laplacian (textbook; the paper's "Fast Poisson Solvers", P:166-168,
P:629).  With S_{jm} = sin(pi j m/(n+1)) (j, m = 1..n) and
λ_m = (4/h^2) sin^2(m pi / (2(n+1)))  (R26),
    u = (2/(n+1))^3  S⊗S⊗S  diag(1/(1/dt + λ_a + λ_b + λ_c))  S⊗S⊗S  q .
Each S⊗S⊗S application is three dense n×n contractions (direct summation, O(n^4)
per solve), no FFT, no folding.  S is built with exact argument reduction
sin(pi ((j m) mod 2(n+1)) / (n+1)).

Independent cross-checks (tests): dense LU of the assembled N^3×N^3 matrix
(``dense_solve``) and explicit stencil application (``apply_operator``).
"""
import numpy as np


def sine_matrix(n: int) -> np.ndarray:
    j = np.arange(1, n + 1)
    arg = np.mod(np.outer(j, j), 2 * (n + 1))
    return np.sin(np.pi * arg / (n + 1))


def eigenvalues(n: int, h: float) -> np.ndarray:
    """λ_m = (4/h^2) sin^2(m pi / (2(n+1))), m = 1..n  (R26; = (2/h^2)(1 - cos(m pi/(n+1))))."""
    m = np.arange(1, n + 1)
    return (4.0 / h ** 2) * np.sin(m * np.pi / (2.0 * (n + 1))) ** 2


def dst3(S: np.ndarray, q: np.ndarray) -> np.ndarray:
    """Apply S along the last three axes of q by direct summation."""
    t = np.tensordot(q, S, axes=([q.ndim - 3], [0]))        # contracts x -> appended last
    t = np.tensordot(t, S, axes=([t.ndim - 3], [0]))        # contracts y
    t = np.tensordot(t, S, axes=([t.ndim - 3], [0]))        # contracts z
    return t  # axis order (…, a, b, c) restored by the three rotations


def solve(q: np.ndarray, h: float, dt: float) -> np.ndarray:
    """u = (I/dt - Δ_h)^{-1} q with zero Dirichlet ghosts, q of shape (..., n, n, n)."""
    n = q.shape[-1]
    S = sine_matrix(n)
    lam = eigenvalues(n, h)
    den = (1.0 / dt + lam[:, None, None]) + lam[None, :, None] + lam[None, None, :]
    qhat = dst3(S, np.asarray(q, dtype=np.float64))
    return (2.0 / (n + 1)) ** 3 * dst3(S, qhat / den)


def apply_operator(u: np.ndarray, h: float, dt: float) -> np.ndarray:
    """(I/dt - Δ_h) u with the 7-point Laplacian and zero ghosts."""
    n = u.shape[-1]
    lead = u.shape[:-3]
    p = np.zeros(lead + (n + 2,) * 3)
    p[..., 1:-1, 1:-1, 1:-1] = u
    c = p[..., 1:-1, 1:-1, 1:-1]
    nb = (p[..., 2:, 1:-1, 1:-1] + p[..., :-2, 1:-1, 1:-1] + p[..., 1:-1, 2:, 1:-1]
          + p[..., 1:-1, :-2, 1:-1] + p[..., 1:-1, 1:-1, 2:] + p[..., 1:-1, 1:-1, :-2])
    return c / dt - (nb - 6.0 * c) / h ** 2


def dense_matrix(n: int, h: float, dt: float) -> np.ndarray:
    """Assembled (I/dt - Δ_h) on the n^3 interior, C-order [x][y][z] unknowns."""
    T = (np.diag(2.0 * np.ones(n)) - np.diag(np.ones(n - 1), 1) - np.diag(np.ones(n - 1), -1)) / h ** 2
    I = np.eye(n)
    return (np.eye(n ** 3) / dt + np.kron(np.kron(T, I), I) + np.kron(np.kron(I, T), I)
            + np.kron(np.kron(I, I), T))


def dense_solve(q: np.ndarray, h: float, dt: float) -> np.ndarray:
    """Brute-force dense LU (numpy.linalg.solve) — only for n <= 12."""
    n = q.shape[-1]
    assert n <= 12
    A = dense_matrix(n, h, dt)
    return np.linalg.solve(A, q.reshape(-1)).reshape(q.shape)
