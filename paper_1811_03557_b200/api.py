"""Thin Python binding over the C ABI (include/dpm.h): argument marshalling only.

Every computation runs in libdpm.so's CUDA kernels.  torch is used for device memory
and streams only.  Names follow the ABI: ``dpm_create`` returns a :class:`DPM` whose
methods are the remaining ``dpm_*`` calls without the prefix.
"""
import ctypes as C

import numpy as np
import torch

from . import _lib as L


def _ptr(t: torch.Tensor):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class _nullctx:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False


def _dev_f64(t: torch.Tensor, name: str):
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous float64 CUDA tensor")
    return t


class DPM:
    """One dpm_ctx: grid + domain + basis + dt on one device."""

    def __init__(self, n, lo, hi, kind="sphere", center=(0.0, 0.0, 0.0), semi=(1.0, 1.0, 1.0), lmax=4,
                 dt=1e-3, basis="cauchy", device=0):
        g = L.Grid(n, lo, hi)
        d = L.Domain(L.SPHERE if kind == "sphere" else L.ELLIPSOID, (C.c_double * 3)(*center),
                     (C.c_double * 3)(*semi))
        if basis not in L.BASES:
            raise ValueError(f"basis must be one of {sorted(L.BASES)}, got {basis!r}")
        b = L.BASES[basis]
        h = C.c_void_p()
        torch.cuda.init()
        L.check(L.lib.dpm_create(C.byref(g), C.byref(d), lmax, dt, b, device, C.byref(h)))
        self._h = h
        self.device = torch.device("cuda", device)
        self.n = n
        self.info = self.query()
        self.K = self.info["K"]

    @classmethod
    def from_config(cls, cfg, device=0):
        return cls(cfg.n, cfg.lo, cfg.hi, cfg.kind, cfg.center, cfg.semi, cfg.lmax, cfg.dt, cfg.basis, device)

    def close(self):
        if getattr(self, "_h", None) and L is not None and getattr(L, "lib", None) is not None:
            L.lib.dpm_destroy(self._h)
        self._h = None

    def __del__(self):
        self.close()

    def _chk(self, st):
        L.check(st, self._h)

    def query(self):
        info = L.Info()
        self._chk(L.lib.dpm_query(self._h, C.byref(info)))
        return {f: getattr(info, f) for f, _ in L.Info._fields_}

    def copy_set(self, which: str) -> np.ndarray:
        key = {"mplus": "n_mplus", "gamma": "n_gamma", "gamma_in": "n_gamma_in", "gamma_ex": "n_gamma_ex",
               "band": "n_band", "nplus": "n_nplus"}[which]
        cnt = self.query()[key]
        out = np.empty(max(cnt, 1), dtype=np.int64)
        self._chk(L.lib.dpm_copy_set(self._h, L.SETS[which], out.ctypes.data_as(C.POINTER(C.c_int64)), cnt))
        return out[:cnt]

    def copy_extension(self):
        i = self.query()
        E = np.empty((i["K"], i["n_gamma"]), dtype=np.float64)   # column-major |γ| x K
        d = np.empty(i["n_gamma"], dtype=np.float64)
        self._chk(L.lib.dpm_copy_extension(self._h, E.ctypes.data_as(L.D), d.ctypes.data_as(L.D)))
        return E.T.copy(), d

    def set_dt(self, dt: float):
        self._chk(L.lib.dpm_set_dt(self._h, dt))

    def set_solver(self, solver: str):
        """"dst3" (3D DST-I) or "dst2_tridiag" (DST-I in x, y + exact tridiagonal solve in z)."""
        self._chk(L.lib.dpm_set_solver(self._h, L.SOLVERS[solver]))
        self.info = self.query()

    def aux_solve_batch(self, q: torch.Tensor, u: torch.Tensor = None, stream=None) -> torch.Tensor:
        _dev_f64(q, "q")
        if u is None:
            u = torch.empty_like(q)
        _dev_f64(u, "u")
        batch = q.numel() // self.n ** 3
        self._chk(L.lib.dpm_aux_solve_batch(self._h, _ptr(q), _ptr(u), batch, _stream(stream)))
        return u

    def set_pass_timing(self, enable: bool):
        self._chk(L.lib.dpm_set_pass_timing(self._h, 1 if enable else 0))

    def pass_times(self):
        """{kind: (ms, launches, points)} for kinds "x", "y", "z" since the last call (synchronizes)."""
        ms = (C.c_double * 3)()
        la = (C.c_int64 * 3)()
        pt = (C.c_int64 * 3)()
        self._chk(L.lib.dpm_pass_times(self._h, ms, la, pt))
        return {k: (ms[i], la[i], pt[i]) for i, k in enumerate(("x", "y", "z"))}

    def aux_solve_batch_host(self, q_host: torch.Tensor, u_host: torch.Tensor = None, stream=None) -> torch.Tensor:
        if q_host.is_cuda or q_host.dtype != torch.float64 or not q_host.is_contiguous():
            raise ValueError("q_host must be a contiguous float64 CPU tensor")
        if u_host is None:
            u_host = torch.empty_like(q_host)
        batch = q_host.numel() // self.n ** 3
        self._chk(L.lib.dpm_aux_solve_batch_host(self._h, _ptr(q_host), _ptr(u_host), batch, _stream(stream)))
        return u_host

    def potential_rhs(self, v_gamma: torch.Tensor, stream=None) -> torch.Tensor:
        """v_gamma: [nrhs, |γ|] (row r = density r) -> q [nrhs, n, n, n]."""
        _dev_f64(v_gamma, "v_gamma")
        nrhs = v_gamma.shape[0]
        q = torch.empty((nrhs, self.n, self.n, self.n), dtype=torch.float64, device=self.device)
        self._chk(L.lib.dpm_potential_rhs(self._h, _ptr(v_gamma), _ptr(q), nrhs, _stream(stream)))
        return q

    def trace(self, u: torch.Tensor, which="gamma", stream=None) -> torch.Tensor:
        _dev_f64(u, "u")
        batch = u.numel() // self.n ** 3
        m = self.info["n_gamma" if which == "gamma" else "n_gamma_in"]
        out = torch.empty((batch, m), dtype=torch.float64, device=self.device)
        self._chk(L.lib.dpm_trace(self._h, _ptr(u), _ptr(out), L.SETS[which], batch, _stream(stream)))
        return out

    def bep_columns(self, c0: int, c1: int, stream=None):
        """Returns (PgE [c1-c0, |γ|], B [c1-c0, |γ_in|]) — row r = column c0+r."""
        i = self.info
        PgE = torch.empty((c1 - c0, i["n_gamma"]), dtype=torch.float64, device=self.device)
        B = torch.empty((c1 - c0, i["n_gamma_in"]), dtype=torch.float64, device=self.device)
        self._chk(L.lib.dpm_bep_columns(self._h, c0, c1, _ptr(PgE), _ptr(B), _stream(stream)))
        return PgE, B

    def bep_factor(self, B: torch.Tensor, stream=None):
        _dev_f64(B, "B")
        self._chk(L.lib.dpm_bep_factor(self._h, _ptr(B), _stream(stream)))

    def build_projection(self, want_outputs=True, stream=None):
        i = self.info
        PgE = B = None
        if want_outputs:
            PgE = torch.empty((self.K, i["n_gamma"]), dtype=torch.float64, device=self.device)
            B = torch.empty((self.K, i["n_gamma_in"]), dtype=torch.float64, device=self.device)
        self._chk(L.lib.dpm_build_projection(self._h, _ptr(PgE), _ptr(B), _stream(stream)))
        return PgE, B

    def boundary_lsq(self, g: torch.Tensor, want_u_gamma=True, stream=None):
        """g: [nrhs, |γ_in|] -> (coef [nrhs, K], u_gamma [nrhs, |γ|])."""
        _dev_f64(g, "g")
        nrhs = g.shape[0]
        coef = torch.empty((nrhs, self.K), dtype=torch.float64, device=self.device)
        ug = torch.empty((nrhs, self.info["n_gamma"]), dtype=torch.float64, device=self.device) if want_u_gamma else None
        self._chk(L.lib.dpm_boundary_lsq(self._h, _ptr(g), _ptr(coef), _ptr(ug), nrhs, _stream(stream)))
        return coef, ug

    def pks_init(self, rho: torch.Tensor, c: torch.Tensor, center, rho_amp, rho_rate, c_amp, c_rate, stream=None,
                 rho_cell_average=False):
        ic = L.PksIC((C.c_double * 3)(*center), rho_amp, rho_rate, c_amp, c_rate, 1 if rho_cell_average else 0)
        self._chk(L.lib.dpm_pks_init(self._h, _ptr(_dev_f64(rho, "rho")), _ptr(_dev_f64(c, "c")), C.byref(ic),
                                     _stream(stream)))

    def pks_diagnostics(self, rho, c, stream=None):
        """{mass, second_moment, free_energy} of a state (dpm_pks_diagnostics)."""
        out = (C.c_double * 3)()
        self._chk(L.lib.dpm_pks_diagnostics(self._h, _ptr(_dev_f64(rho, "rho")), _ptr(_dev_f64(c, "c")), out,
                                            _stream(stream)))
        return {"mass": out[0], "second_moment": out[1], "free_energy": out[2]}

    def pks_step(self, rho, c, nsteps, chi=1.0, dt_cap=1e-4, dt_rule=0, clamp=1, stream=None, coupling=0):
        prm = L.PksParams(chi, dt_cap, dt_rule, clamp, coupling)
        logs = (L.StepLog * max(nsteps, 1))()
        self._chk(L.lib.dpm_pks_step(self._h, _ptr(_dev_f64(rho, "rho")), _ptr(_dev_f64(c, "c")), nsteps,
                                     C.byref(prm), logs, _stream(stream)))
        return [{f: getattr(logs[i], f) for f, _ in L.StepLog._fields_} for i in range(nsteps)]


def dpm_create(n, lo, hi, kind, center, semi, lmax, dt, basis, device=0) -> DPM:
    return DPM(n, lo, hi, kind, center, semi, lmax, dt, basis, device)


def dpm_aux_solve_batch(ctx: DPM, q, u=None, stream=None):
    return ctx.aux_solve_batch(q, u, stream)


def dpm_build_projection(ctx: DPM, stream=None):
    return ctx.build_projection(True, stream)


def dpm_boundary_lsq(ctx: DPM, g, stream=None):
    return ctx.boundary_lsq(g, True, stream)


def dpm_pks_step(ctx: DPM, rho, c, nsteps, **kw):
    return ctx.pks_step(rho, c, nsteps, **kw)


class Octant(DPM):
    """One config-5 octant subdomain (dpm_create_octant): canonical frame, box [lo, hi]^3."""

    def __init__(self, n, lo, hi, octant, radius=1.0, lmax_cap=12, deg_if=12, dt=1e-5, device=0):
        g = L.Grid(n, lo, hi)
        h = C.c_void_p()
        torch.cuda.init()
        L.check(L.lib.dpm_create_octant(C.byref(g), octant, radius, lmax_cap, deg_if, dt, device, C.byref(h)))
        self._h = h
        self.device = torch.device("cuda", device)
        self.n = n
        self.octant = octant
        self.info = self.query()
        rows = C.c_int64()
        K = C.c_int32()
        self._chk(L.lib.dpm_dd_info(self._h, C.byref(rows), C.byref(K)))
        self.n_rows, self.K = rows.value, K.value

    def copy_assign(self) -> np.ndarray:
        out = np.empty(max(self.info["n_gamma"], 1), dtype=np.uint8)
        self._chk(L.lib.dpm_dd_copy_assign(self._h, out.ctypes.data_as(C.POINTER(C.c_uint8))))
        return out[: self.info["n_gamma"]]

    def _t(self, *shape):
        return torch.empty(shape, dtype=torch.float64, device=self.device)

    def bep_block(self, want=False, stream=None):
        B = self._t(self.K, self.n_rows) if want else None       # row c = column c of B_s
        self._chk(L.lib.dpm_dd_bep_block(self._h, _ptr(B), _stream(stream)))
        return B

    def bep_block_from(self, ref, want=False, stream=None):
        """B_s = B_ref diag(S_s) from another octant of the same geometry (dpm_dd_bep_block_from)."""
        B = self._t(self.K, self.n_rows) if want else None
        self._chk(L.lib.dpm_dd_bep_block_from(self._h, ref._h, _ptr(B), _stream(stream)))
        return B

    def colnorm2(self, stream=None):
        out = self._t(self.K)
        self._chk(L.lib.dpm_dd_colnorm2(self._h, _ptr(out), _stream(stream)))
        return out

    def gram(self, pass_, nrm2_sum=None, stream=None):
        G = self._t(self.K, self.K)
        self._chk(L.lib.dpm_dd_gram(self._h, pass_, _ptr(nrm2_sum), _ptr(G), _stream(stream)))
        return G

    def chol(self, pass_, G_sum, stream=None):
        self._chk(L.lib.dpm_dd_chol(self._h, pass_, _ptr(_dev_f64(G_sum, "G_sum")), _stream(stream)))

    # phase-level step (batched AP solves across octants; see include/dpm.h)
    def dd_rhs(self, rho, c, chi, fq, stream=None):
        self._chk(L.lib.dpm_dd_rhs(self._h, _ptr(_dev_f64(rho, "rho")), _ptr(_dev_f64(c, "c")), chi,
                                   _ptr(_dev_f64(fq, "fq")), _stream(stream)))

    def dd_lsq_rhs(self, wk, stream=None):
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            y = self._t(2, self.K)
        self._chk(L.lib.dpm_dd_lsq_rhs(self._h, _ptr(_dev_f64(wk, "wk")), _ptr(y), _stream(stream)))
        return y

    def dd_lsq_rhs_shared(self, octs, wk, stream=None):
        """Σ_s M_s g_s over octant contexts of one device sharing the canonical geometry (this one first):
        one pass over this octant's Q (dpm_dd_lsq_rhs_shared); wk: [noct][2][n][n][n]."""
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            y = self._t(2, self.K)
        arr = (C.c_void_p * len(octs))(*[o._h.value for o in octs])
        self._chk(L.lib.dpm_dd_lsq_rhs_shared(arr, len(octs), _ptr(_dev_f64(wk, "wk")), _ptr(y), _stream(stream)))
        return y

    def dd_green_rhs_shared(self, octs, coef, clamp, fq, wk, stream=None):
        """dd_green_rhs for octant contexts of one device sharing the canonical geometry: one basis
        evaluation per γ point for all of them (dpm_dd_green_rhs_shared); fq, wk: [noct][2][n][n][n]."""
        arr = (C.c_void_p * len(octs))(*[o._h.value for o in octs])
        self._chk(L.lib.dpm_dd_green_rhs_shared(arr, len(octs), _ptr(_dev_f64(coef, "C")), clamp, _ptr(_dev_f64(fq, "fq")),
                                                _ptr(_dev_f64(wk, "wk")), _stream(stream)))

    def dd_green_rhs(self, C, clamp, fq, wk, stream=None):
        self._chk(L.lib.dpm_dd_green_rhs(self._h, _ptr(_dev_f64(C, "C")), clamp, _ptr(_dev_f64(fq, "fq")),
                                         _ptr(_dev_f64(wk, "wk")), _stream(stream)))

    def dd_restrict(self, wk, rho, c, stream=None):
        self._chk(L.lib.dpm_dd_restrict(self._h, _ptr(_dev_f64(wk, "wk")), _ptr(_dev_f64(rho, "rho")),
                                        _ptr(_dev_f64(c, "c")), _stream(stream)))

    def chol_copy(self, pass_, src: "Octant", stream=None):
        """The same CholeskyQR pass from `src` (same device, same summed Gram, already factored)."""
        self._chk(L.lib.dpm_dd_chol_copy(self._h, pass_, src._h, _stream(stream)))

    def dd_pks_init(self, rho, c, center, rho_amp, rho_rate, c_amp, c_rate, stream=None, rho_cell_average=0):
        ic = L.PksIC((C.c_double * 3)(*center), rho_amp, rho_rate, c_amp, c_rate, int(rho_cell_average))
        self._chk(L.lib.dpm_dd_pks_init(self._h, _ptr(_dev_f64(rho, "rho")), _ptr(_dev_f64(c, "c")), C.byref(ic),
                                        _stream(stream)))

    def cfl(self, c, chi=1.0, stream=None) -> float:
        out = C.c_double()
        self._chk(L.lib.dpm_dd_cfl(self._h, _ptr(_dev_f64(c, "c")), chi, C.byref(out), _stream(stream)))
        return out.value

    def cfl_async(self, c, chi=1.0, stream=None):
        self._chk(L.lib.dpm_dd_cfl(self._h, _ptr(_dev_f64(c, "c")), chi, None, _stream(stream)))

    def cfl_result(self, chi=1.0, stream=None) -> float:
        out = C.c_double()
        self._chk(L.lib.dpm_dd_cfl_result(self._h, chi, C.byref(out), _stream(stream)))
        return out.value

    def stats(self, stream=None):
        st = (C.c_double * 6)()
        self._chk(L.lib.dpm_dd_stats(self._h, st, _stream(stream)))
        return {"mass": st[0], "rho_max": st[1], "rho_min": st[2], "c_min": st[3], "nonfinite": st[4],
                "rho_max_mplus": st[5]}

    def local_finish_async(self, Cglob, rho, c, clamp=1, stream=None):
        self._chk(L.lib.dpm_dd_local_finish(self._h, _ptr(_dev_f64(Cglob, "C")), clamp, _ptr(rho), _ptr(c), None,
                                            _stream(stream)))

    def local_begin(self, rho, c, chi=1.0, stream=None):
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            y = self._t(2, self.K)
        self._chk(L.lib.dpm_dd_local_begin(self._h, _ptr(rho), _ptr(c), chi, _ptr(y), _stream(stream)))
        return y

    def local_finish(self, Cglob, rho, c, clamp=1, stream=None):
        st = (C.c_double * 6)()
        self._chk(L.lib.dpm_dd_local_finish(self._h, _ptr(_dev_f64(Cglob, "C")), clamp, _ptr(rho), _ptr(c), st,
                                            _stream(stream)))
        return {"mass": st[0], "rho_max": st[1], "rho_min": st[2], "c_min": st[3], "nonfinite": st[4],
                "rho_max_mplus": st[5]}


class CaseOneSubdomain(Octant):
    """One subdomain of the paper's two-subdomain DD, Case 1 (dpm_create_dd1, NEXT-3): sub 0 = Ω1, the
    ball r1; sub 1 = Ω2, the shell r1 < |x| < r2; grid (n, lo, hi) its own auxiliary cube.  Every
    dpm_dd_* method of Octant applies."""

    def __init__(self, n, lo, hi, sub, r1=0.25, r2=0.5, mz=0, mg=0, dt=1e-8, device=0):
        g = L.Grid(n, lo, hi)
        h = C.c_void_p()
        torch.cuda.init()
        L.check(L.lib.dpm_create_dd1(C.byref(g), sub, r1, r2, mz, mg, dt, device, C.byref(h)))
        self._h = h
        self.device = torch.device("cuda", device)
        self.n = n
        self.sub = sub
        self.info = self.query()
        rows = C.c_int64()
        K = C.c_int32()
        self._chk(L.lib.dpm_dd_info(self._h, C.byref(rows), C.byref(K)))
        self.n_rows, self.K = rows.value, K.value
