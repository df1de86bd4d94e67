"""ctypes declarations of libdpm.so (include/dpm.h).  Argument marshalling only.

There is no fallback: if libdpm.so is missing or fails to load, importing this module
raises (build it with ``python -m paper_1811_03557_b200.build`` or ``__graft_entry__.build()``).
"""
import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdpm.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libdpm.so not built at {LIB_PATH}; run python -m paper_1811_03557_b200.build")
lib = C.CDLL(LIB_PATH)

DPM_OK, DPM_ERR_INVALID, DPM_ERR_OOM, DPM_ERR_CUDA, DPM_ERR_STATE, DPM_ERR_RANK, DPM_ERR_NONFINITE = range(7)
STATUS = {0: "DPM_OK", 1: "DPM_ERR_INVALID", 2: "DPM_ERR_OOM", 3: "DPM_ERR_CUDA", 4: "DPM_ERR_STATE",
          5: "DPM_ERR_RANK", 6: "DPM_ERR_NONFINITE"}
SPHERE, ELLIPSOID = 0, 1
BASIS_CAUCHY, BASIS_NEUMANN0, BASIS_CAUCHY_ZONAL, BASIS_NEUMANN0_ZONAL = 0, 1, 2, 3
BASIS_NEUMANN0_2TERM, BASIS_NEUMANN0_2TERM_ZONAL = 4, 5
BASES = {"cauchy": BASIS_CAUCHY, "neumann0": BASIS_NEUMANN0,
         "cauchy_zonal": BASIS_CAUCHY_ZONAL, "neumann0_zonal": BASIS_NEUMANN0_ZONAL,
         "neumann0_2term": BASIS_NEUMANN0_2TERM, "neumann0_2term_zonal": BASIS_NEUMANN0_2TERM_ZONAL}
SOLVER_DST3, SOLVER_DST2_TRIDIAG = 0, 1
SOLVERS = {"dst3": SOLVER_DST3, "dst2_tridiag": SOLVER_DST2_TRIDIAG}
SETS = {"mplus": 0, "gamma": 1, "gamma_in": 2, "gamma_ex": 3, "band": 4, "nplus": 5}
MAX_N = 128


class Grid(C.Structure):
    _fields_ = [("n", C.c_int32), ("lo", C.c_double), ("hi", C.c_double)]


class Domain(C.Structure):
    _fields_ = [("kind", C.c_int32), ("center", C.c_double * 3), ("semi", C.c_double * 3)]


class Info(C.Structure):
    _fields_ = [("n", C.c_int32), ("K", C.c_int32), ("lmax", C.c_int32), ("basis", C.c_int32),
                ("h", C.c_double), ("dt", C.c_double),
                ("n_mplus", C.c_int64), ("n_gamma", C.c_int64), ("n_gamma_in", C.c_int64),
                ("n_gamma_ex", C.c_int64), ("n_band", C.c_int64), ("n_nplus", C.c_int64),
                ("ghosts_in_nplus", C.c_int64), ("have_projection", C.c_int32), ("bep_cond_est", C.c_double),
                ("solver", C.c_int32), ("n_exact_ties", C.c_int64), ("n_exact_ties_inside", C.c_int64)]


class PksIC(C.Structure):
    _fields_ = [("center", C.c_double * 3), ("rho_amp", C.c_double), ("rho_rate", C.c_double),
                ("c_amp", C.c_double), ("c_rate", C.c_double), ("rho_cell_average", C.c_int32)]


class PksParams(C.Structure):
    _fields_ = [("chi", C.c_double), ("dt_cap", C.c_double), ("dt_rule", C.c_int32), ("clamp", C.c_int32),
                ("coupling", C.c_int32)]


class StepLog(C.Structure):
    _fields_ = [("t", C.c_double), ("dt", C.c_double), ("mass", C.c_double), ("rho_max", C.c_double),
                ("rho_min", C.c_double), ("c_min", C.c_double), ("rebuilt", C.c_int32), ("step", C.c_int32),
                ("rho_max_mplus", C.c_double), ("clamp_max", C.c_double), ("lsq_resid", C.c_double)]


P = C.c_void_p
D = C.POINTER(C.c_double)
_sig = {
    "dpm_create": ([C.POINTER(Grid), C.POINTER(Domain), C.c_int32, C.c_double, C.c_int32, C.c_int32,
                    C.POINTER(P)], C.c_int),
    "dpm_destroy": ([P], None),
    "dpm_query": ([P, C.POINTER(Info)], C.c_int),
    "dpm_last_error": ([P], C.c_char_p),
    "dpm_copy_set": ([P, C.c_int32, C.POINTER(C.c_int64), C.c_int64], C.c_int),
    "dpm_copy_extension": ([P, D, D], C.c_int),
    "dpm_set_dt": ([P, C.c_double], C.c_int),
    "dpm_aux_solve_batch": ([P, P, P, C.c_int64, P], C.c_int),
    "dpm_set_solver": ([P, C.c_int32], C.c_int),
    "dpm_aux_solve_batch_host": ([P, P, P, C.c_int64, P], C.c_int),
    "dpm_potential_rhs": ([P, P, P, C.c_int32, P], C.c_int),
    "dpm_trace": ([P, P, P, C.c_int32, C.c_int64, P], C.c_int),
    "dpm_bep_columns": ([P, C.c_int32, C.c_int32, P, P, P], C.c_int),
    "dpm_bep_factor": ([P, P, P], C.c_int),
    "dpm_build_projection": ([P, P, P, P], C.c_int),
    "dpm_boundary_lsq": ([P, P, P, P, C.c_int32, P], C.c_int),
    "dpm_pks_init": ([P, P, P, C.POINTER(PksIC), P], C.c_int),
    "dpm_pks_diagnostics": ([P, P, P, C.POINTER(C.c_double), P], C.c_int),
    "dpm_pks_step": ([P, P, P, C.c_int32, C.POINTER(PksParams), C.POINTER(StepLog), P], C.c_int),
    "dpm_launch_count": ([], C.c_int64),
    "dpm_set_pass_timing": ([P, C.c_int32], C.c_int),
    "dpm_create_octant": ([C.POINTER(Grid), C.c_int32, C.c_double, C.c_int32, C.c_int32, C.c_double, C.c_int32,
                           C.POINTER(P)], C.c_int),
    "dpm_create_dd1": ([C.POINTER(Grid), C.c_int32, C.c_double, C.c_double, C.c_int32, C.c_int32, C.c_double,
                        C.c_int32, C.POINTER(P)], C.c_int),
    "dpm_dd_info": ([P, C.POINTER(C.c_int64), C.POINTER(C.c_int32)], C.c_int),
    "dpm_dd_copy_assign": ([P, C.POINTER(C.c_uint8)], C.c_int),
    "dpm_dd_bep_block": ([P, P, P], C.c_int),
    "dpm_dd_bep_block_from": ([P, P, P, P], C.c_int),
    "dpm_dd_colnorm2": ([P, P, P], C.c_int),
    "dpm_dd_gram": ([P, C.c_int32, P, P, P], C.c_int),
    "dpm_dd_chol": ([P, C.c_int32, P, P], C.c_int),
    "dpm_dd_chol_copy": ([P, C.c_int32, P, P], C.c_int),
    "dpm_dd_rhs": ([P, P, P, C.c_double, P, P], C.c_int),
    "dpm_dd_lsq_rhs": ([P, P, P, P], C.c_int),
    "dpm_dd_lsq_rhs_shared": ([C.POINTER(P), C.c_int32, P, P, P], C.c_int),
    "dpm_dd_green_rhs": ([P, P, C.c_int32, P, P, P], C.c_int),
    "dpm_dd_green_rhs_shared": ([C.POINTER(P), C.c_int32, P, C.c_int32, P, P, P], C.c_int),
    "dpm_dd_restrict": ([P, P, P, P, P], C.c_int),
    "dpm_dd_pks_init": ([P, P, P, C.POINTER(PksIC), P], C.c_int),
    "dpm_dd_cfl": ([P, P, C.c_double, D, P], C.c_int),
    "dpm_dd_cfl_result": ([P, C.c_double, D, P], C.c_int),
    "dpm_dd_stats": ([P, D, P], C.c_int),
    "dpm_dd_local_begin": ([P, P, P, C.c_double, P, P], C.c_int),
    "dpm_dd_local_finish": ([P, P, C.c_int32, P, P, D, P], C.c_int),
    "dpm_pass_times": ([P, D, C.POINTER(C.c_int64), C.POINTER(C.c_int64)], C.c_int),
}
EXPORTED = tuple(_sig)
for _name, (_args, _res) in _sig.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res


class DPMError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def check(status, ctx=None):
    if status != DPM_OK:
        msg = lib.dpm_last_error(ctx)
        raise DPMError(status, msg.decode() if msg else "")
