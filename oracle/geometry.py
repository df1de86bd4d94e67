"""Boundary geometry for gamma points — oracle (test infrastructure only).

For each gamma point p the extension operator (`eqn:extension_operator`)
needs: the orthogonal projection (foot) p' on Γ, the signed distance d (positive
outside, along the outward normal), and the angles (θ, φ) of the foot for
the spherical-harmonic basis.

* sphere: foot = c + r (p - c)/|p - c|, d = |p - c| - r, angles of (p - c).
* ellipsoid: foot = the closest point of the ellipsoid; it solves
  x_i = s_i^2 p_i / (s_i^2 + t) with F(t) = Σ (s_i p_i / (s_i^2 + t))^2 - 1 = 0.
  F is strictly decreasing on (-min s_i^2, ∞); the root is found by plain
  bisection to machine precision.  d = sign(t) |p - foot|.  Angles are the
  parametric angles of the unit vector (x'/a, y'/b, z'/c).
Returned ``unit`` is the unit vector whose spherical angles (θ, φ) feed sh.real_sh.
"""
import numpy as np


def sphere_geometry(P: np.ndarray, center, r: float):
    v = P - np.asarray(center)[None, :]
    rad = np.sqrt((v ** 2).sum(axis=1))
    unit = v / rad[:, None]
    foot = np.asarray(center)[None, :] + r * unit
    d = rad - r
    return foot, d, unit


def _ellipsoid_t(p: np.ndarray, s: np.ndarray) -> float:
    def F(t):
        return float(((s * p / (s ** 2 + t)) ** 2).sum() - 1.0)

    lo = -float((s ** 2).min()) * (1.0 - 1e-12)
    hi = 1.0
    while F(hi) > 0.0:
        hi *= 2.0
    if F(lo) < 0.0:   # degenerate: root pinned at the axis; not reached for gamma points
        raise ValueError("ellipsoid foot: point on the medial axis")
    for _ in range(400):
        mid = 0.5 * (lo + hi)
        if mid == lo or mid == hi:
            break
        if F(mid) > 0.0:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def ellipsoid_geometry(P: np.ndarray, center, semi):
    s = np.asarray(semi, dtype=np.float64)
    c = np.asarray(center, dtype=np.float64)
    feet = np.empty_like(P)
    d = np.empty(P.shape[0])
    unit = np.empty_like(P)
    for k in range(P.shape[0]):
        p = P[k] - c
        t = _ellipsoid_t(p, s)
        x = s ** 2 * p / (s ** 2 + t)
        feet[k] = x + c
        d[k] = np.sign(t) * np.sqrt(((p - x) ** 2).sum())
        u = x / s
        unit[k] = u / np.sqrt((u ** 2).sum())
    return feet, d, unit


def geometry(P: np.ndarray, kind: str, center, semi):
    if kind == "sphere":
        return sphere_geometry(P, center, semi[0])
    if kind == "ellipsoid":
        return ellipsoid_geometry(P, center, semi)
    raise ValueError(kind)
