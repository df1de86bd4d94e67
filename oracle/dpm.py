"""Difference Potentials Method operators — oracle (test infrastructure only).

Literal definitions, column by column (no fusion, no batching tricks):
* particular solution G f (`rhs:particular_solution`): AP with q = f on M+,
  0 on M-, restricted to N+.  ABI scaling (R4): q = f/dt.
* difference potential P_{N+γ} v_γ (Def. `DP`): AP with q = 0 on M+ and
  L[v_γ] on M-, v_γ zero-extended off γ.  ABI scaling: q = (I/dt - Δ_h)[v_γ] on M-.
* trace Tr_γ, Tr_γin and P_γ = Tr_γ P_{N+γ}.
* extension operator with spectral Cauchy data:
  columns c = comp*(L+1)^2 + ν (R9): comp 0 -> Y_ν(foot);
  comp 1 -> d Y_ν ("cauchy", 2-term u, du/dn) or (d^2/2) Y_ν ("neumann0");
  "*_zonal": Y_ν replaced by the paper's zonal modes P_l^0(cos θ), l = 0..L, K = 2 (L+1);
  "neumann0_2term[_zonal]": the 2-term extension (β = 0) with ∂u/∂n = 0, comp 0 only.
* reduced BEP (`eqn:BEP_recast` P:287-290): B = Tr_γin (E - P_γ E).
* least squares: numpy.linalg.lstsq (SVD) and an independent plain
  Householder QR (``householder_lstsq``) used as a cross-check.
* discrete generalized Green's formula: u = P_{N+γ} u_γ + G f on N+.
"""
import numpy as np

from . import ap, geometry, grid, sh


def gamma_points(g: grid.Grid, ps: grid.PointSets) -> np.ndarray:
    idx = ps.list("gamma")
    n = g.n
    i, j, k = np.unravel_index(idx, (n, n, n))
    x = g.coords()
    return np.stack([x[i], x[j], x[k]], axis=1)


def extension_matrix(g, ps, kind, center, semi, lmax, basis):
    """E (|γ| × K), K = 2 (L+1)^2 (full real SH) or 2 (L+1) (zonal), plus (d, unit) of
    the gamma points."""
    P = gamma_points(g, ps)
    foot, d, unit = geometry.geometry(P, kind, center, semi)
    Y = sh.zonal(lmax, unit) if basis.endswith("_zonal") else sh.real_sh(lmax, unit)
    if basis in ("neumann0_2term", "neumann0_2term_zonal"):   # β = 0 with ∂u/∂n = 0: π = u|Γ
        return Y, d, unit, foot
    if basis in ("cauchy", "cauchy_zonal"):
        second = d[:, None] * Y
    elif basis in ("neumann0", "neumann0_zonal"):
        second = 0.5 * (d ** 2)[:, None] * Y
    else:
        raise ValueError(basis)
    return np.concatenate([Y, second], axis=1), d, unit, foot


def scatter(values: np.ndarray, idx: np.ndarray, n: int) -> np.ndarray:
    """Zero-extend values given on a flat-index list to the n^3 box."""
    out = np.zeros(n ** 3)
    out[idx] = values
    return out.reshape(n, n, n)


def potential_rhs(v_gamma: np.ndarray, g, ps, dt: float) -> np.ndarray:
    """q = χ_{M-} (I/dt - Δ_h)[v_γ]  (Def. DP, scaled per R4)."""
    V = scatter(v_gamma, ps.list("gamma"), g.n)
    q = ap.apply_operator(V, g.h, dt)
    q[ps.mplus] = 0.0
    return q


def particular_rhs(f_mplus_box: np.ndarray, ps, dt: float) -> np.ndarray:
    """q = χ_{M+} f / dt  (scaled per R4)."""
    q = np.where(ps.mplus, f_mplus_box, 0.0) / dt
    return q


def potential_columns(E: np.ndarray, g, ps, dt: float, chunk: int = 32) -> np.ndarray:
    """u_c = AP solve of potential_rhs(E[:, c]) for every column, shape (K, n, n, n).  The columns are
    independent; they are solved `chunk` at a time only to bound the host memory of the batch."""
    K = E.shape[1]
    U = np.empty((K, g.n, g.n, g.n))
    for c0 in range(0, K, chunk):
        Q = np.stack([potential_rhs(E[:, c], g, ps, dt) for c in range(c0, min(K, c0 + chunk))])
        U[c0:c0 + len(Q)] = ap.solve(Q, g.h, dt)
    return U


def potential_trace(E: np.ndarray, g, ps, dt: float, idx: np.ndarray, chunk: int = 16) -> np.ndarray:
    """Tr_idx of potential_columns(E): (len(idx), K), without holding all K boxes (large n)."""
    K = E.shape[1]
    out = np.empty((len(idx), K))
    for c0 in range(0, K, chunk):
        c1 = min(K, c0 + chunk)
        out[:, c0:c1] = trace(potential_columns(E[:, c0:c1], g, ps, dt, 1 if g.n >= 64 else chunk), idx).T
    return out


def trace(U: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """Tr on a flat-index list; U is (..., n, n, n) -> (..., len(idx))."""
    lead = U.shape[:-3]
    return U.reshape(lead + (-1,))[..., idx]


def projection_and_bep(E, g, ps, dt):
    """P_γE (|γ|×K) and B = Tr_γin(E - P_γ E) (|γ_in|×K)."""
    U = potential_columns(E, g, ps, dt)
    PgE = trace(U, ps.list("gamma")).T
    gin_pos = np.searchsorted(ps.list("gamma"), ps.list("gamma_in"))
    B = E[gin_pos] - PgE[gin_pos]
    return PgE, B, U


def full_projection(g, ps, dt):
    """The full |γ|×|γ| matrix P_γ (one AP solve per γ point; test artefact, R11)."""
    ng = len(ps.list("gamma"))
    return projection_and_bep(np.eye(ng), g, ps, dt)[0]


def lstsq(B: np.ndarray, rhs: np.ndarray) -> np.ndarray:
    return np.linalg.lstsq(B, rhs, rcond=None)[0]


def householder_lstsq(B: np.ndarray, rhs: np.ndarray) -> np.ndarray:
    """Plain Householder QR without pivoting ("QR decomposition"), then R^{-1} Q^T rhs."""
    A = np.array(B, dtype=np.float64)
    b = np.array(rhs, dtype=np.float64)
    m, k = A.shape
    for j in range(k):
        x = A[j:, j]
        alpha = -np.copysign(np.linalg.norm(x), x[0])
        v = x.copy()
        v[0] -= alpha
        vn = np.linalg.norm(v)
        if vn == 0.0:
            continue
        v /= vn
        A[j:, j:] -= 2.0 * np.outer(v, v @ A[j:, j:])
        b[j:] -= 2.0 * np.outer(v, v @ b[j:]).reshape(b[j:].shape)
    R = np.triu(A[:k, :k])
    y = b[:k]
    C = np.zeros_like(y)
    for i in range(k - 1, -1, -1):
        C[i] = (y[i] - R[i, i + 1:] @ C[i + 1:]) / R[i, i]
    return C


def green(u_gamma: np.ndarray, f_box: np.ndarray, g, ps, dt: float) -> np.ndarray:
    """Generalized Green's formula evaluated as ONE AP solve of the combined
    right-hand side χ_{M+} f/dt + χ_{M-}(I/dt - Δ_h)[u_γ] (R20), restricted to N+."""
    q = particular_rhs(f_box, ps, dt) + potential_rhs(u_gamma, g, ps, dt)
    u = ap.solve(q, g.h, dt)
    return np.where(ps.nplus, u, 0.0)


def green_two_solve(u_gamma, f_box, g, ps, dt):
    """P_{N+γ} u_γ + G f with two separate solves (the literal P:306 form; test cross-check)."""
    up = ap.solve(potential_rhs(u_gamma, g, ps, dt), g.h, dt)
    uf = ap.solve(particular_rhs(f_box, ps, dt), g.h, dt)
    return np.where(ps.nplus, up + uf, 0.0)


def cfg1_outputs(cfg):
    """R11: U (K+1 solves), P_γE, B, C = lstsq(B, U_particular[γ_in]) for config 1."""
    from dpm_inputs import cfg1_particular_values
    g, ps = grid.point_sets_for(cfg)
    E, d, unit, foot = extension_matrix(g, ps, cfg.kind, cfg.center, cfg.semi, cfg.lmax, cfg.basis)
    PgE, B, Ub = projection_and_bep(E, g, ps, cfg.dt)
    qp = scatter(cfg1_particular_values(int(ps.mplus.sum())), ps.list("mplus"), g.n)
    up = ap.solve(qp, g.h, cfg.dt)
    gvec = trace(up, ps.list("gamma_in"))
    C = lstsq(B, gvec)
    U = np.concatenate([Ub, up[None]], axis=0)
    return dict(g=g, ps=ps, E=E, PgE=PgE, B=B, C=C, U=U, q_particular=qp, rhs=gvec)
