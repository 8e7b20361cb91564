"""ctypes binding of libchebmg_b200.so (include/chebmg_b200.h).

The product path has no fallback: if the native library is missing this module
raises ImportError with the build command, and every numeric call goes through
the CUDA library (there is no CPU implementation in this package).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CMG_LIB") or os.path.join(_HERE, "lib", "libchebmg_b200.so")  # CMG_LIB: A/B builds
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "chebmg_b200.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"chebmg_b200 native library not built: {LIB_PATH} is missing. "
        "Run `make lib` (or __graft_entry__.build()) first; there is no CPU fallback."
    )

lib = C.CDLL(LIB_PATH)

dp = C.POINTER(C.c_double)
vp = C.c_void_p
sz = C.c_size_t
u64 = C.c_uint64

CMG_OK, CMG_EINVAL, CMG_ERANGE, CMG_ERUNTIME, CMG_ECUDA, CMG_ENCCL = range(6)


class CmgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class ChebConfig(C.Structure):
    _fields_ = [("family", C.c_int), ("lambda_tilde", C.c_double),
                ("lambda_max_multiplier", C.c_double), ("lambda_min_multiplier", C.c_double)]


class CycleConfigC(C.Structure):
    _fields_ = [("smoother", ChebConfig), ("k_pre", sz), ("k_post", sz)]


class SolveOptionsC(C.Structure):
    _fields_ = [("tol", C.c_double), ("maxit", sz), ("restart", sz),
                ("reorthogonalize", C.c_int), ("enforce_spd_preconditioner", C.c_int)]


class SolveReportC(C.Structure):
    _fields_ = [("iterations", sz), ("fine_matvecs", sz), ("rho", C.c_double),
                ("converged", C.c_int), ("status", C.c_char * 128), ("wall_time_sec", C.c_double),
                ("residual_history", dp), ("history_capacity", sz), ("history_len", sz)]


class SemDesc(C.Structure):
    _fields_ = [("order", C.c_int), ("ex", C.c_int), ("ey", C.c_int), ("ez", C.c_int),
                ("geometry", C.c_int), ("eps", C.c_double), ("rank", C.c_int), ("nranks", C.c_int)]


PRECOND_FN = C.CFUNCTYPE(None, vp, vp, vp)

_protos = {
    "cmg_last_error": (C.c_char_p, []),
    "cmg_version": (C.c_char_p, []),
    "cmg_ctx_create": (C.c_int, [C.c_int, vp, C.POINTER(vp)]),
    "cmg_ctx_destroy": (C.c_int, [vp]),
    "cmg_ctx_synchronize": (C.c_int, [vp]),
    "cmg_ctx_kernel_launches": (u64, [vp]),
    "cmg_malloc": (C.c_int, [vp, sz, C.POINTER(vp)]),
    "cmg_free": (C.c_int, [vp, vp]),
    "cmg_upload": (C.c_int, [vp, vp, vp, sz]),
    "cmg_download": (C.c_int, [vp, vp, vp, sz]),
    "cmg_random_vector_host": (C.c_int, [sz, u64, dp]),
    "cmg_dot": (C.c_int, [vp, sz, vp, vp, dp]),
    "cmg_norm2": (C.c_int, [vp, sz, vp, dp]),
    "cmg_axpy": (C.c_int, [vp, sz, C.c_double, vp, vp]),
    "cmg_fd_op_create": (C.c_int, [vp, sz, C.c_double, C.c_double, C.POINTER(vp)]),
    "cmg_op_destroy": (C.c_int, [vp]),
    "cmg_op_rows": (sz, [vp]),
    "cmg_op_vec_len": (sz, [vp]),
    "cmg_op_apply": (C.c_int, [vp, vp, vp]),
    "cmg_op_diagonal": (C.c_int, [vp, vp]),
    "cmg_op_applications": (sz, [vp]),
    "cmg_op_reset_applications": (None, [vp]),
    "cmg_fd_build_problem_host": (C.c_int, [sz, C.c_double, C.c_double, u64, dp, dp]),
    "cmg_jacobi_inverse_diagonal": (C.c_int, [vp, sz, vp, vp]),
    "cmg_estimate_lambda_max": (C.c_int, [vp, vp, sz, u64, dp]),
    "cmg_chebyshev_smooth": (C.c_int, [vp, vp, C.POINTER(ChebConfig), sz, vp, vp, C.c_int]),
    "cmg_beta_coefficients": (C.c_int, [sz, dp]),
    "cmg_fd_hierarchy_create": (C.c_int, [vp, sz, C.c_double, C.c_double, sz, sz, u64, C.POINTER(vp)]),
    "cmg_fd_hierarchy_clone": (C.c_int, [vp, vp, C.POINTER(vp)]),
    "cmg_fd_hierarchy_destroy": (C.c_int, [vp]),
    "cmg_fd_hierarchy_lambda_tilde": (C.c_double, [vp]),
    "cmg_fd_hierarchy_op": (vp, [vp]),
    "cmg_fd_hierarchy_inv_diag": (vp, [vp]),
    "cmg_fd_hierarchy_coarse_dim": (sz, [vp]),
    "cmg_fd_prolong": (C.c_int, [vp, vp, vp]),
    "cmg_fd_restrict": (C.c_int, [vp, vp, vp]),
    "cmg_fd_coarse_solve": (C.c_int, [vp, vp, vp]),
    "cmg_fd_v_cycle": (C.c_int, [vp, C.POINTER(CycleConfigC), vp, vp, C.c_int]),
    "cmg_fd_estimate_C": (C.c_int, [vp, sz, C.c_uint64, C.c_int, C.POINTER(C.c_double),
                                    C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(sz)]),
    "cmg_fd_preconditioner_apply": (C.c_int, [vp, C.POINTER(CycleConfigC), vp, vp]),
    "cmg_precond_fd_vcycle": (C.c_int, [vp, C.POINTER(CycleConfigC), C.POINTER(vp)]),
    "cmg_precond_identity": (C.c_int, [vp, C.POINTER(vp)]),
    "cmg_precond_callback": (C.c_int, [vp, PRECOND_FN, vp, C.POINTER(vp)]),
    "cmg_precond_destroy": (C.c_int, [vp]),
    "cmg_precond_apply": (C.c_int, [vp, vp, vp]),
    "cmg_pcg": (C.c_int, [vp, vp, vp, vp, vp, C.POINTER(SolveOptionsC), C.POINTER(SolveReportC)]),
    "cmg_pgmres": (C.c_int, [vp, vp, vp, vp, vp, C.POINTER(SolveOptionsC), C.POINTER(SolveReportC)]),
    "cmg_stationary_solve": (C.c_int, [vp, vp, vp, C.c_double, sz, vp, C.POINTER(SolveReportC)]),
    "cmg_sem_op_create": (C.c_int, [vp, C.POINTER(SemDesc), C.POINTER(vp)]),
    "cmg_sem_partition": (C.c_int, [C.POINTER(SemDesc), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "cmg_sem_slot_map_host": (C.c_int, [C.POINTER(SemDesc), C.POINTER(C.c_int64)]),
    "cmg_sem_gs_map_host": (C.c_int, [C.POINTER(SemDesc), C.POINTER(C.c_int64)]),
    "cmg_sem_local_slots": (sz, [C.POINTER(SemDesc)]),
    "cmg_sem_rhs": (C.c_int, [vp, vp]),
    "cmg_sem_basis_host": (C.c_int, [C.c_int, vp, vp, vp]),
    "cmg_sem_interp_host": (C.c_int, [C.c_int, C.c_int, vp]),
    "cmg_sem_fdm1d_host": (C.c_int, [C.c_int, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                                     C.c_int, vp, vp]),
    "cmg_pmg_create": (C.c_int, [vp, C.POINTER(SemDesc), C.c_int, C.POINTER(C.c_int), C.c_int, sz, u64,
                                 C.POINTER(vp)]),
    "cmg_pmg_destroy": (C.c_int, [vp]),
    "cmg_pmg_op": (vp, [vp, C.c_int]),
    "cmg_pmg_lambda_tilde": (C.c_double, [vp, C.c_int]),
    "cmg_pmg_inv_diag": (vp, [vp, C.c_int]),
    "cmg_pmg_prolong": (C.c_int, [vp, C.c_int, vp, vp]),
    "cmg_pmg_restrict": (C.c_int, [vp, C.c_int, vp, vp]),
    "cmg_pmg_coarse_solve": (C.c_int, [vp, vp, vp]),
    "cmg_pmg_schwarz_apply": (C.c_int, [vp, C.c_int, vp, vp]),
    "cmg_pmg_smooth": (C.c_int, [vp, C.c_int, C.POINTER(ChebConfig), sz, vp, vp, C.c_int]),
    "cmg_pmg_v_cycle": (C.c_int, [vp, C.POINTER(CycleConfigC), vp, vp, C.c_int]),
    "cmg_precond_pmg": (C.c_int, [vp, C.POINTER(CycleConfigC), C.POINTER(vp)]),
    "cmg_nccl_unique_id": (C.c_int, [C.POINTER(C.c_ubyte)]),
    "cmg_ctx_attach_nccl": (C.c_int, [vp, C.POINTER(C.c_ubyte), C.c_int, C.c_int]),
}

missing = []
for _name, (_res, _args) in _protos.items():
    try:
        _f = getattr(lib, _name)
    except AttributeError:
        missing.append(_name)
        continue
    _f.restype = _res
    _f.argtypes = _args


def check(rc: int) -> None:
    if rc != CMG_OK:
        msg = lib.cmg_last_error().decode(errors="replace")
        if rc == CMG_EINVAL:
            raise ValueError(msg)
        if rc == CMG_ERANGE:
            raise IndexError(msg)
        raise CmgError(rc, msg)


def header_symbols() -> list[str]:
    """Function names declared in include/chebmg_b200.h."""
    import re

    text = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"\b(cmg_[a-z0-9_]+)\s*\(", text)) - {"cmg_precond_fn"})
