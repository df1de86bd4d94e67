"""Real orthonormal spherical harmonics — oracle (test infrastructure only).

Basis of the spectral approximation (`eqn:spectral_approximation_sd`);
BASELINE.json asks for the full real SH of degree <= L:
  Y_l0  = N_l0 P_l(cos θ)
  Y_lm  = sqrt(2) N_lm P_l^m(cos θ) cos(m φ)        m > 0
  Y_l,-m = sqrt(2) N_lm P_l^m(cos θ) sin(m φ)       m > 0
  N_lm  = sqrt((2l+1)/(4 pi) (l-m)!/(l+m)!),  P_l^m WITHOUT the Condon-Shortley phase.
Index ν = l^2 + l + m.  θ = arccos(u_z), φ = atan2(u_y, u_x) of the unit vector u.
P_l^m by the textbook three-term recurrence in l at fixed m.
"""
import math

import numpy as np


def assoc_legendre(lmax: int, x: np.ndarray) -> np.ndarray:
    """P[l][m] (m <= l) without Condon-Shortley phase, shape (lmax+1, lmax+1, len(x))."""
    x = np.asarray(x, dtype=np.float64)
    s = np.sqrt(np.maximum(0.0, 1.0 - x * x))
    P = np.zeros((lmax + 1, lmax + 1) + x.shape)
    for m in range(lmax + 1):
        # P_m^m = (2m-1)!! s^m
        dfact = 1.0
        for k in range(1, 2 * m, 2):
            dfact *= k
        P[m, m] = dfact * s ** m
        if m + 1 <= lmax:
            P[m + 1, m] = x * (2 * m + 1) * P[m, m]
        for l in range(m + 2, lmax + 1):
            P[l, m] = ((2 * l - 1) * x * P[l - 1, m] - (l + m - 1) * P[l - 2, m]) / (l - m)
    return P


def zonal(lmax: int, unit: np.ndarray) -> np.ndarray:
    """phi[:, l] = P_l^0(cos θ), l = 0..lmax (the zonal modes, unnormalised Legendre
    polynomials of cos θ = u_z), by Bonnet's recurrence (l+1) P_{l+1} = (2l+1) x P_l - l P_{l-1}."""
    x = np.clip(np.asarray(unit, dtype=np.float64)[:, 2], -1.0, 1.0)
    P = np.zeros((x.shape[0], lmax + 1))
    P[:, 0] = 1.0
    if lmax >= 1:
        P[:, 1] = x
    for l in range(1, lmax):
        P[:, l + 1] = ((2 * l + 1) * x * P[:, l] - l * P[:, l - 1]) / (l + 1)
    return P


def real_sh(lmax: int, unit: np.ndarray) -> np.ndarray:
    """Y[:, ν] for ν = l^2 + l + m, shape (npts, (lmax+1)^2)."""
    u = np.asarray(unit, dtype=np.float64)
    theta = np.arccos(np.clip(u[:, 2], -1.0, 1.0))
    phi = np.arctan2(u[:, 1], u[:, 0])
    P = assoc_legendre(lmax, np.cos(theta))
    Y = np.zeros((u.shape[0], (lmax + 1) ** 2))
    for l in range(lmax + 1):
        for m in range(0, l + 1):
            N = math.sqrt((2 * l + 1) / (4 * math.pi) * math.factorial(l - m) / math.factorial(l + m))
            if m == 0:
                Y[:, l * l + l] = N * P[l, 0]
            else:
                Y[:, l * l + l + m] = math.sqrt(2.0) * N * P[l, m] * np.cos(m * phi)
                Y[:, l * l + l - m] = math.sqrt(2.0) * N * P[l, m] * np.sin(m * phi)
    return Y
