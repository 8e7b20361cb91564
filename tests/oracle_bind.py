"""ctypes bindings of the test-only checkers: oracle/liboracle.so (C restatement)
and oracle/_ref/libchebmg_ref.so (the compiled, unmodified reference).

Test infrastructure only -- the product package never imports this.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libchebmg_ref.so")

dp = C.POINTER(C.c_double)
sz = C.c_size_t


def P(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(dp)


class _Rep(C.Structure):
    _fields_ = [("iterations", sz), ("fine_matvecs", sz), ("rho", C.c_double), ("converged", C.c_int),
                ("status", C.c_char * 128), ("wall", C.c_double), ("hist_len", sz)]


class _Cfg(C.Structure):
    _fields_ = [("Lx", C.c_double), ("n", sz), ("factor", sz), ("family", C.c_int), ("k", sz),
                ("cycle", C.c_int), ("driver", C.c_int), ("tol", C.c_double), ("restart", sz),
                ("maxit", sz), ("rhs_seed", C.c_uint64), ("eigen_seed", C.c_uint64),
                ("tuning_seed", C.c_uint64), ("lmaxm", C.c_double), ("lminm", C.c_double),
                ("eig_it", sz)]


class _Res(C.Structure):
    _fields_ = [("report", _Rep), ("lambda_tilde", C.c_double), ("tuned", C.c_double)]


class _CCfg(C.Structure):
    _fields_ = [("family", C.c_int), ("lambda_tilde", C.c_double), ("lmaxm", C.c_double),
                ("lminm", C.c_double)]


@dataclass
class Report:
    iterations: int
    fine_matvecs: int
    history: list
    converged: bool
    status: str
    rho: float = 1.0
    lambda_tilde: float = float("nan")
    tuned_lambda_min: float | None = None
    wall_time_sec: float = 0.0
    x: np.ndarray | None = field(default=None, repr=False)


_orc = None


def oracle():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            raise FileNotFoundError(f"{ORACLE_SO} missing: run `make -C oracle`")
        L = C.CDLL(ORACLE_SO)
        L.orc_fd_hier_create.restype = C.c_void_p
        L.orc_fd_hier_create.argtypes = [sz, C.c_double, C.c_double, sz, sz, C.c_uint64]
        L.orc_fd_hier_lambda_tilde.restype = C.c_double
        L.orc_fd_hier_lambda_tilde.argtypes = [C.c_void_p]
        L.orc_fd_hier_destroy.argtypes = [C.c_void_p]
        L.orc_fd_hier_op.restype = C.c_void_p
        L.orc_fd_hier_op.argtypes = [C.c_void_p]
        L.orc_fd_hier_coarse_dim.restype = sz
        L.orc_fd_hier_coarse_dim.argtypes = [C.c_void_p]
        L.orc_fd_hier_bandwidth.restype = sz
        L.orc_fd_hier_bandwidth.argtypes = [C.c_void_p]
        L.orc_fd_hier_coarse_solve.argtypes = [C.c_void_p, dp, dp]
        L.orc_fd_v_cycle.argtypes = [C.c_void_p, C.POINTER(_CCfg), sz, sz, dp, dp, C.c_int]
        L.orc_fd_run_case_with.argtypes = [C.POINTER(_Cfg), C.c_void_p, dp, dp, C.POINTER(_Res)]
        L.orc_chebyshev_smooth.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(_CCfg), sz, dp, dp, C.c_int]
        L.orc_random_vector.argtypes = [sz, C.c_uint64, dp]
        L.orc_fd_build_problem.argtypes = [sz, C.c_double, C.c_double, C.c_uint64, dp, dp]
        L.orc_fd_stencil_apply.argtypes = [sz, C.c_double, C.c_double, dp, dp]
        L.orc_fd_prolong.argtypes = [sz, sz, dp, dp]
        L.orc_fd_restrict.argtypes = [sz, sz, dp, dp]
        L.orc_beta_coefficients.restype = dp
        L.orc_beta_coefficients.argtypes = [sz]
        L.orc_dot.restype = C.c_double
        L.orc_dot.argtypes = [sz, dp, dp]
        _orc = L
    return _orc


_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        L = C.CDLL(REF_SO)
        L.ref_hier_create.restype = C.c_void_p
        L.ref_hier_create.argtypes = [sz, C.c_double, C.c_double, sz, sz, C.c_uint64]
        L.ref_hier_destroy.argtypes = [C.c_void_p]
        L.ref_hier_lambda.restype = C.c_double
        L.ref_hier_lambda.argtypes = [C.c_void_p]
        L.ref_hier_bandwidth.restype = sz
        L.ref_hier_bandwidth.argtypes = [C.c_void_p]
        L.ref_hier_coarse_nnz.restype = sz
        L.ref_hier_coarse_nnz.argtypes = [C.c_void_p]
        L.ref_hier_coarse_solve.argtypes = [C.c_void_p, dp, dp]
        L.ref_hier_coarse_apply.argtypes = [C.c_void_p, dp, dp]
        L.ref_random_vector.argtypes = [sz, C.c_uint64, dp]
        L.ref_dot.restype = C.c_double
        L.ref_dot.argtypes = [sz, dp, dp]
        L.ref_fd_build_problem.argtypes = [sz, C.c_double, C.c_double, C.c_uint64, dp, dp]
        L.ref_fd_stencil_apply.argtypes = [sz, C.c_double, C.c_double, dp, dp]
        L.ref_fd_prolong.argtypes = [sz, sz, dp, dp]
        L.ref_fd_restrict.argtypes = [sz, sz, dp, dp]
        L.ref_smooth.argtypes = [C.c_void_p, C.c_int, sz, C.c_double, C.c_double, C.c_double, dp, dp,
                                 C.c_int, C.POINTER(sz)]
        L.ref_v_cycle.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double, sz, sz, dp, dp, C.c_int,
                                  C.POINTER(sz)]
        L.ref_solve.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double, sz, sz, dp, dp,
                                C.c_double, sz, sz, dp, dp, sz, C.POINTER(sz), C.POINTER(sz),
                                C.POINTER(sz), C.POINTER(C.c_int), C.c_char_p, C.POINTER(C.c_double),
                                C.POINTER(C.c_double)]
        L.ref_run_case_with.argtypes = [C.c_void_p, C.c_double, sz, sz, C.c_int, sz, C.c_int, C.c_int,
                                        C.c_double, sz, sz, dp, sz, C.POINTER(sz), C.POINTER(sz),
                                        C.POINTER(sz), C.POINTER(C.c_int), C.c_char_p,
                                        C.POINTER(C.c_double), C.POINTER(C.c_double),
                                        C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.ref_estimate_C.restype = C.c_double
        L.ref_estimate_C.argtypes = [C.c_void_p, sz, C.c_uint64]
        L.ref_last_error.restype = C.c_char_p
        _ref = L
    return _ref


# ---------------------------------------------------------------- oracle helpers
def random_vector(n: int, seed: int) -> np.ndarray:
    out = np.empty(n)
    oracle().orc_random_vector(n, seed, P(out))
    return out


def build_problem(n: int, Lx: float, Ly: float, seed: int):
    m = (n - 1) ** 2
    u, b = np.empty(m), np.empty(m)
    oracle().orc_fd_build_problem(n, Lx, Ly, seed, P(u), P(b))
    return u, b


def stencil_apply(n: int, Lx: float, Ly: float, x: np.ndarray) -> np.ndarray:
    y = np.empty_like(x)
    oracle().orc_fd_stencil_apply(n, Lx, Ly, P(x), P(y))
    return y


class OracleHierarchy:
    def __init__(self, n: int, Lx: float, factor: int, Ly: float = 1.0, eig_iters: int = 30, seed: int = 7):
        self.n, self.Lx, self.Ly, self.factor = n, Lx, Ly, factor
        self.h = oracle().orc_fd_hier_create(n, Lx, Ly, factor, eig_iters, seed)
        if not self.h:
            raise ValueError("build_hierarchy: factor must divide n")
        self.lambda_tilde = oracle().orc_fd_hier_lambda_tilde(self.h)
        self.nf = (n - 1) ** 2
        self.nc = oracle().orc_fd_hier_coarse_dim(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            oracle().orc_fd_hier_destroy(self.h)

    def coarse_solve(self, rc: np.ndarray) -> np.ndarray:
        ec = np.empty_like(rc)
        oracle().orc_fd_hier_coarse_solve(self.h, P(rc), P(ec))
        return ec

    def smooth(self, family: int, order: int, b: np.ndarray, x: np.ndarray, x_is_zero: bool,
               lmaxm: float = 1.03, lminm: float = 0.1, lambda_tilde: float | None = None) -> np.ndarray:
        """chebyshev_smooth on the hierarchy's operator; returns the new x."""
        L = oracle()
        x = x.copy()
        cfg = _CCfg(family, self.lambda_tilde if lambda_tilde is None else lambda_tilde, lmaxm, lminm)
        # orc_smoother {inv_diag, NULL, NULL}: inv_diag is constant 1/c
        c = 2.0 * (1.0 / (self.Lx / self.n) ** 2 + 1.0 / (self.Ly / self.n) ** 2)
        invd = np.full(self.nf, 1.0 / c)

        class _Sm(C.Structure):
            _fields_ = [("inv_diag", dp), ("S_apply", C.c_void_p), ("S_ctx", C.c_void_p)]

        sm = _Sm(P(invd), None, None)
        rc = L.orc_chebyshev_smooth(L.orc_fd_hier_op(self.h), C.byref(sm), C.byref(cfg), order, P(b), P(x),
                                    1 if x_is_zero else 0)
        if rc == -1:
            raise ValueError("ChebyshevConfig invalid")
        if rc == -2:
            raise IndexError("beta order out of range")
        return x

    def v_cycle(self, family: int, k_pre: int, k_post: int, b: np.ndarray, x: np.ndarray, x_is_zero: bool,
                lmaxm: float = 1.03, lminm: float = 0.1) -> np.ndarray:
        x = x.copy()
        cfg = _CCfg(family, self.lambda_tilde, lmaxm, lminm)
        oracle().orc_fd_v_cycle(self.h, C.byref(cfg), k_pre, k_post, P(b), P(x), 1 if x_is_zero else 0)
        return x

    def run_case(self, family: int, k: int, cycle: int, driver: int, tol: float = 1e-6, restart: int = 30,
                 maxit: int = 500, lmaxm: float = 1.03, lminm: float = 0.1) -> Report:
        cfg = _Cfg(self.Lx, self.n, self.factor, family, k, cycle, driver, tol, restart, maxit, 1234, 7, 4321,
                   lmaxm, lminm, 30)
        hist = np.zeros(maxit + 2)
        x = np.zeros(self.nf)
        res = _Res()
        rc = oracle().orc_fd_run_case_with(C.byref(cfg), self.h, P(hist), P(x), C.byref(res))
        if rc != 0:
            raise ValueError(f"run_case failed ({rc})")
        r = res.report
        return Report(int(r.iterations), int(r.fine_matvecs), hist[: r.hist_len].tolist(), bool(r.converged),
                      r.status.decode(), float(r.rho), float(res.lambda_tilde),
                      None if math.isnan(res.tuned) else float(res.tuned), float(r.wall), x)


class RefHierarchy:
    """The compiled reference (oracle/_ref), same surface as OracleHierarchy."""

    def __init__(self, n: int, Lx: float, factor: int, Ly: float = 1.0, eig_iters: int = 30, seed: int = 7):
        self.n, self.Lx, self.Ly, self.factor = n, Lx, Ly, factor
        self.h = ref().ref_hier_create(n, Lx, Ly, factor, eig_iters, seed)
        if not self.h:
            raise ValueError(ref().ref_last_error().decode())
        self.lambda_tilde = ref().ref_hier_lambda(self.h)
        self.nf = (n - 1) ** 2

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_hier_destroy(self.h)

    def run_case(self, family: int, k: int, cycle: int, driver: int, tol: float = 1e-6, restart: int = 30,
                 maxit: int = 500) -> Report:
        hist = np.zeros(maxit + 2)
        hl, its, mv = sz(), sz(), sz()
        cv = C.c_int()
        st = C.create_string_buffer(128)
        rho, wall, lam, tl = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        rc = ref().ref_run_case_with(self.h, self.Lx, self.n, self.factor, family, k, cycle, driver, tol, restart,
                                     maxit, P(hist), maxit + 2, C.byref(hl), C.byref(its), C.byref(mv),
                                     C.byref(cv), st, C.byref(rho), C.byref(wall), C.byref(lam), C.byref(tl))
        if rc != 0:
            raise ValueError(ref().ref_last_error().decode())
        return Report(its.value, mv.value, hist[: hl.value].tolist(), bool(cv.value), st.value.decode(), rho.value,
                      lam.value, None if tl.value < 0 else tl.value, wall.value)

    def smooth(self, family: int, order: int, b: np.ndarray, x: np.ndarray, x_is_zero: bool,
               lmaxm: float = 1.03, lminm: float = 0.1, lambda_tilde: float | None = None):
        x = x.copy()
        apps = sz()
        rc = ref().ref_smooth(self.h, family, order, self.lambda_tilde if lambda_tilde is None else lambda_tilde,
                              lmaxm, lminm, P(b), P(x), 1 if x_is_zero else 0, C.byref(apps))
        if rc == 1:
            raise ValueError(ref().ref_last_error().decode())
        if rc == 2:
            raise IndexError(ref().ref_last_error().decode())
        return x, apps.value

    def v_cycle(self, family: int, k_pre: int, k_post: int, b: np.ndarray, x: np.ndarray, x_is_zero: bool,
                lmaxm: float = 1.03, lminm: float = 0.1):
        x = x.copy()
        apps = sz()
        ref().ref_v_cycle(self.h, family, lmaxm, lminm, k_pre, k_post, P(b), P(x), 1 if x_is_zero else 0,
                          C.byref(apps))
        return x, apps.value


def hexs(xs) -> list[str]:
    return [float(v).hex() for v in xs]


def unhex(xs) -> np.ndarray:
    return np.array([float.fromhex(s) for s in xs])


# ---------------------------------------------------------------- SEM (restated spec; parity unpinned)
def _sem_protos(L):
    L.orc_sem_create.restype = C.c_void_p
    L.orc_sem_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double]
    L.orc_sem_destroy.argtypes = [C.c_void_p]
    L.orc_sem_n.restype = sz
    L.orc_sem_n.argtypes = [C.c_void_p]
    L.orc_sem_op.restype = C.c_void_p
    L.orc_sem_op.argtypes = [C.c_void_p]
    L.orc_op_apply.argtypes = [C.c_void_p, dp, dp]
    L.orc_sem_diagonal.argtypes = [C.c_void_p, dp]
    L.orc_sem_rhs.argtypes = [C.c_void_p, dp]
    L.orc_sem_local_to_global_map.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
    L.orc_sem_geom.argtypes = [C.c_void_p, dp, dp]
    L.orc_sem_prolong.argtypes = [C.c_void_p, C.c_void_p, dp, dp]
    L.orc_sem_restrict.argtypes = [C.c_void_p, C.c_void_p, dp, dp]
    L.orc_sem_schwarz.argtypes = [C.c_void_p, C.c_int, dp, dp]
    L.orc_gll.argtypes = [C.c_int, dp, dp]
    L.orc_deriv_matrix.argtypes = [C.c_int, dp, dp]
    L.orc_interp_matrix.argtypes = [C.c_int, C.c_int, dp]
    L.orc_pmg_create.restype = C.c_void_p
    L.orc_pmg_create.argtypes = [C.c_int, C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                 C.c_int, sz, C.c_uint64]
    L.orc_pmg_destroy.argtypes = [C.c_void_p]
    L.orc_pmg_op.restype = C.c_void_p
    L.orc_pmg_op.argtypes = [C.c_void_p, C.c_int]
    L.orc_pmg_sem.restype = C.c_void_p
    L.orc_pmg_sem.argtypes = [C.c_void_p, C.c_int]
    L.orc_pmg_lambda_tilde.restype = C.c_double
    L.orc_pmg_lambda_tilde.argtypes = [C.c_void_p, C.c_int]
    L.orc_pmg_v_cycle.restype = C.c_int
    L.orc_pmg_v_cycle.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double, sz, sz, dp, dp, C.c_int]
    L.orc_pmg_coarse_solve.argtypes = [C.c_void_p, dp, dp]
    L.orc_pmg_solve.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double, sz, sz, dp, C.c_double, sz,
                                sz, dp, dp, C.POINTER(_Rep)]
    L.orc_chebyshev_smooth.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(_CCfg), sz, dp, dp, C.c_int]
    L.orc_estimate_lambda_max.restype = C.c_double
    L.orc_estimate_lambda_max.argtypes = [C.c_void_p, C.c_void_p, sz, C.c_uint64]


class _Smoother(C.Structure):
    _fields_ = [("inv_diag", dp), ("S_apply", C.c_void_p), ("S_ctx", C.c_void_p)]


class OracleSem:
    """Restated SEM operator on one level (canonical interior ordering)."""

    def __init__(self, N, ex, ey, ez, geometry=0, eps=1.0, lib=None):
        self.L = lib or oracle()
        _sem_protos(self.L)
        self.N, self.ex, self.ey, self.ez = N, ex, ey, ez
        self.s = self.L.orc_sem_create(N, ex, ey, ez, geometry, eps)
        if not self.s:
            raise ValueError("orc_sem_create failed")
        self.n = self.L.orc_sem_n(self.s)
        self._own = True

    def __del__(self):
        if getattr(self, "_own", False) and self.s:
            self.L.orc_sem_destroy(self.s)

    def apply(self, x):
        y = np.empty(self.n)
        self.L.orc_op_apply(self.L.orc_sem_op(self.s), P(np.ascontiguousarray(x)), P(y))
        return y

    def diagonal(self):
        d = np.empty(self.n)
        self.L.orc_sem_diagonal(self.s, P(d))
        return d

    def rhs(self):
        b = np.empty(self.n)
        self.L.orc_sem_rhs(self.s, P(b))
        return b

    def gs_map(self):
        m = np.empty(self.ex * self.ey * self.ez * (self.N + 1) ** 3, dtype=np.int64)
        self.L.orc_sem_local_to_global_map(self.s, m.ctypes.data_as(C.POINTER(C.c_int64)))
        return m

    def geom(self):
        E, NP = self.ex * self.ey * self.ez, (self.N + 1) ** 3
        G, B = np.empty(E * 6 * NP), np.empty(E * NP)
        self.L.orc_sem_geom(self.s, P(G), P(B))
        return G, B

    def schwarz(self, r, ras):
        out = np.empty(self.n)
        self.L.orc_sem_schwarz(self.s, 1 if ras else 0, P(np.ascontiguousarray(r)), P(out))
        return out


def gll(N):
    xi, w = np.empty(N + 1), np.empty(N + 1)
    L = oracle()
    _sem_protos(L)
    L.orc_gll(N, P(xi), P(w))
    D = np.empty((N + 1) ** 2)
    L.orc_deriv_matrix(N, P(xi), P(D))
    return xi, w, D.reshape(N + 1, N + 1)


def interp_matrix(Nf, Nc):
    L = oracle()
    _sem_protos(L)
    J = np.empty((Nf + 1) * (Nc + 1))
    L.orc_interp_matrix(Nf, Nc, P(J))
    return J.reshape(Nf + 1, Nc + 1)


class OraclePmg:
    """Restated p-multigrid hierarchy; `lib` may be the _ref library (reference templates)."""

    def __init__(self, orders, ex, ey, ez, geometry=0, eps=1.0, smoother=0, eig_iters=30, seed=7, lib=None):
        self.L = lib or oracle()
        _sem_protos(self.L)
        self.orders = list(orders)
        arr = (C.c_int * len(orders))(*orders)
        self.p = self.L.orc_pmg_create(len(orders), arr, ex, ey, ez, geometry, eps, smoother, eig_iters, seed)
        if not self.p:
            raise ValueError("orc_pmg_create failed")
        self.lambda_tilde = [self.L.orc_pmg_lambda_tilde(self.p, l) for l in range(len(orders))]
        self.n = [self.L.orc_sem_n(self.L.orc_pmg_sem(self.p, l)) for l in range(len(orders))]

    def __del__(self):
        if getattr(self, "p", None):
            self.L.orc_pmg_destroy(self.p)

    def sem(self, level):
        s = OracleSem.__new__(OracleSem)
        s.L = self.L
        s.s = self.L.orc_pmg_sem(self.p, level)
        s.n = self.n[level]
        s._own = False
        return s

    def v_cycle(self, family, kpre, kpost, b, lmaxm=1.03, lminm=0.1):
        x = np.zeros(self.n[0])
        rc = self.L.orc_pmg_v_cycle(self.p, family, lmaxm, lminm, kpre, kpost, P(np.ascontiguousarray(b)), P(x), 1)
        assert rc == 0
        return x

    def coarse_solve(self, rc):
        e = np.empty_like(rc)
        self.L.orc_pmg_coarse_solve(self.p, P(np.ascontiguousarray(rc)), P(e))
        return e

    def prolong(self, level, xc):
        y = np.empty(self.n[level])
        self.L.orc_sem_prolong(self.L.orc_pmg_sem(self.p, level), self.L.orc_pmg_sem(self.p, level + 1),
                               P(np.ascontiguousarray(xc)), P(y))
        return y

    def restrict(self, level, xf):
        y = np.empty(self.n[level + 1])
        self.L.orc_sem_restrict(self.L.orc_pmg_sem(self.p, level), self.L.orc_pmg_sem(self.p, level + 1),
                                P(np.ascontiguousarray(xf)), P(y))
        return y

    def smooth(self, level, family, order, b, x, x_is_zero, lmaxm=1.03, lminm=0.1, inv_diag=None):
        s = self.sem(level)
        invd = 1.0 / s.diagonal() if inv_diag is None else inv_diag
        sm = _Smoother(P(invd), None, None)
        cfg = _CCfg(family, self.lambda_tilde[level], lmaxm, lminm)
        x = np.array(x, dtype=np.float64)
        rc = self.L.orc_chebyshev_smooth(self.L.orc_pmg_op(self.p, level), C.byref(sm), C.byref(cfg), order,
                                         P(np.ascontiguousarray(b)), P(x), 1 if x_is_zero else 0)
        assert rc == 0
        return x

    def solve(self, driver, family, kpre, kpost, b, tol=1e-8, maxit=500, restart=30, lmaxm=1.03, lminm=0.1):
        x = np.zeros(self.n[0])
        hist = np.zeros(maxit + 2)
        rep = _Rep()
        self.L.orc_pmg_solve(self.p, driver, family, lmaxm, lminm, kpre, kpost, P(np.ascontiguousarray(b)), tol,
                             maxit, restart, P(x), P(hist), C.byref(rep))
        return Report(int(rep.iterations), int(rep.fine_matvecs), hist[: rep.hist_len].tolist(), bool(rep.converged),
                      rep.status.decode(), float(rep.rho), wall_time_sec=float(rep.wall), x=x)


def ref_sem_solve(pmg: OraclePmg, driver, family, kpre, kpost, b, tol=1e-8, maxit=500, restart=30):
    """The reference's own pcg/pgmres templates driving the restated SEM operator
    (oracle/ref_driver.cpp); `pmg` must have been created with lib=ref()."""
    R = ref()
    R.ref_sem_solve.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double, sz, sz, dp, C.c_double, sz,
                                sz, dp, dp, sz, C.POINTER(sz), C.POINTER(sz), C.POINTER(sz), C.POINTER(C.c_int),
                                C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    x = np.zeros(pmg.n[0])
    hist = np.zeros(maxit + 2)
    hl, its, mv = sz(), sz(), sz()
    cv = C.c_int()
    st = C.create_string_buffer(128)
    rho, wall = C.c_double(), C.c_double()
    rc = R.ref_sem_solve(pmg.p, driver, family, 1.03, 0.1, kpre, kpost, P(np.ascontiguousarray(b)), tol, maxit,
                         restart, P(x), P(hist), maxit + 2, C.byref(hl), C.byref(its), C.byref(mv), C.byref(cv), st,
                         C.byref(rho), C.byref(wall))
    assert rc == 0, R.ref_last_error()
    return Report(its.value, mv.value, hist[: hl.value].tolist(), bool(cv.value), st.value.decode(), rho.value,
                  wall_time_sec=wall.value, x=x)


class RefPmg:
    """p-MG on the reference's own templates (oracle/ref_driver.cpp RefPmg):
    pgmres/pcg, chebyshev_smooth, residual_into, estimate_lambda_max and the
    BandedCholesky coarse solve; SEM levels, diagonals and transfers from the
    restatement."""

    def __init__(self, orders, ex, ey, ez, geometry=0, eps=1.0, smoother=0, eig_iters=30, seed=7):
        R = ref()
        _sem_protos(R)
        R.ref_pmg_create.restype = C.c_void_p
        R.ref_pmg_create.argtypes = [C.c_int, C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                     C.c_int, sz, C.c_uint64]
        R.ref_pmg_destroy.argtypes = [C.c_void_p]
        R.ref_pmg_levels.restype = C.c_void_p
        R.ref_pmg_levels.argtypes = [C.c_void_p]
        R.ref_pmg_lambda.restype = C.c_double
        R.ref_pmg_lambda.argtypes = [C.c_void_p, C.c_int]
        R.ref_pmg_coarse_bandwidth.restype = sz
        R.ref_pmg_coarse_bandwidth.argtypes = [C.c_void_p]
        R.ref_pmg_coarse_solve.argtypes = [C.c_void_p, dp, dp]
        R.ref_pmg_v_cycle.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double, sz, sz, dp, dp]
        R.ref_pmg_smooth.argtypes = [C.c_void_p, C.c_int, C.c_int, sz, C.c_double, C.c_double, dp, dp, C.c_int,
                                     C.POINTER(sz)]
        R.ref_pmg_solve.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double, sz, sz, dp, C.c_double,
                                    sz, sz, dp, dp, sz, C.POINTER(sz), C.POINTER(sz), C.POINTER(sz),
                                    C.POINTER(C.c_int), C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        self.R = R
        self.L = R
        self.orders = list(orders)
        arr = (C.c_int * len(orders))(*orders)
        self.h = R.ref_pmg_create(len(orders), arr, ex, ey, ez, geometry, eps, smoother, eig_iters, seed)
        if not self.h:
            raise ValueError(R.ref_last_error().decode())
        self.p = R.ref_pmg_levels(self.h)
        self.lambda_tilde = [R.ref_pmg_lambda(self.h, l) for l in range(len(orders))]
        self.n = [R.orc_sem_n(R.orc_pmg_sem(self.p, l)) for l in range(len(orders))]

    def __del__(self):
        if getattr(self, "h", None):
            self.R.ref_pmg_destroy(self.h)

    def sem(self, level):
        return OraclePmg.sem(self, level)

    def prolong(self, level, xc):
        return OraclePmg.prolong(self, level, xc)

    def restrict(self, level, xf):
        return OraclePmg.restrict(self, level, xf)

    def coarse_solve(self, rc):
        e = np.empty_like(rc)
        assert self.R.ref_pmg_coarse_solve(self.h, P(np.ascontiguousarray(rc)), P(e)) == 0
        return e

    def v_cycle(self, family, kpre, kpost, b, lmaxm=1.03, lminm=0.1):
        x = np.zeros(self.n[0])
        rc = self.R.ref_pmg_v_cycle(self.h, family, lmaxm, lminm, kpre, kpost, P(np.ascontiguousarray(b)), P(x))
        assert rc == 0, self.R.ref_last_error()
        return x

    def smooth(self, level, family, order, b, x, x_is_zero, lmaxm=1.03, lminm=0.1):
        x = np.array(x, dtype=np.float64)
        apps = sz()
        rc = self.R.ref_pmg_smooth(self.h, level, family, order, lmaxm, lminm, P(np.ascontiguousarray(b)), P(x),
                                   1 if x_is_zero else 0, C.byref(apps))
        assert rc == 0, self.R.ref_last_error()
        return x, apps.value

    def solve(self, driver, family, kpre, kpost, b, tol=1e-8, maxit=500, restart=30, lmaxm=1.03, lminm=0.1):
        x = np.zeros(self.n[0])
        hist = np.zeros(maxit + 2)
        hl, its, mv = sz(), sz(), sz()
        cv = C.c_int()
        st = C.create_string_buffer(128)
        rho, wall = C.c_double(), C.c_double()
        rc = self.R.ref_pmg_solve(self.h, driver, family, lmaxm, lminm, kpre, kpost, P(np.ascontiguousarray(b)),
                                  tol, maxit, restart, P(x), P(hist), maxit + 2, C.byref(hl), C.byref(its),
                                  C.byref(mv), C.byref(cv), st, C.byref(rho), C.byref(wall))
        assert rc == 0, self.R.ref_last_error()
        return Report(its.value, mv.value, hist[: hl.value].tolist(), bool(cv.value), st.value.decode(), rho.value,
                      wall_time_sec=wall.value, x=x)


# ---------------------------------------------------------------- reference-side binding
ADAPTER_SO = os.path.join(ROOT, "oracle", "_ref", "libchebmg_adapter.so")
_ad = None


def adapter_available() -> bool:
    return os.path.exists(ADAPTER_SO)


def adapter():
    """oracle/_ref/libchebmg_adapter.so: integration/chebmg_b200_adapter.hpp compiled
    against the unmodified reference headers (oracle/adapter_driver.cpp entry points)."""
    global _ad
    if _ad is None:
        L = C.CDLL(ADAPTER_SO)
        out = [dp, sz, C.POINTER(sz), C.POINTER(sz), C.POINTER(sz), C.POINTER(C.c_int), C.c_char_p]
        L.ad_last_error.restype = C.c_char_p
        L.ad_fd_smooth.argtypes = [sz, C.c_double, C.c_int, sz, C.c_double, dp, dp, C.c_int, C.POINTER(sz)]
        L.ad_fd_solve_templates.argtypes = [sz, C.c_double, sz, C.c_int, sz, sz, C.c_int, C.c_double, dp] + out
        L.ad_fd_run_case_b200.argtypes = [sz, C.c_double, sz, C.c_int, sz, C.c_int, C.c_int, C.c_double] + out + [
            C.POINTER(C.c_double)]
        L.ad_pmg_create.restype = C.c_void_p
        L.ad_pmg_create.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int]
        L.ad_pmg_destroy.argtypes = [C.c_void_p]
        L.ad_pmg_lambda.restype = C.c_double
        L.ad_pmg_lambda.argtypes = [C.c_void_p, C.c_int]
        L.ad_pmg_smooth.argtypes = [C.c_void_p, C.c_int, sz, C.c_double, dp, dp, C.c_int, C.POINTER(sz)]
        L.ad_pmg_solve.argtypes = [C.c_void_p, C.c_int, C.c_int, sz, sz, dp, C.c_double, dp] + out
        _ad = L
    return _ad


def adapter_report(fn, *args, maxit=500, n=0, extra=()):
    """Call an adapter solve entry point (trailing outputs: hist, cap, len, its, mv, cv, status)."""
    x = np.zeros(n)
    hist = np.zeros(maxit + 2)
    hl, its, mv = sz(), sz(), sz()
    cv = C.c_int()
    st = C.create_string_buffer(128)
    head = list(args) + ([P(x)] if n else [])
    rc = fn(*head, P(hist), maxit + 2, C.byref(hl), C.byref(its), C.byref(mv), C.byref(cv), st, *extra)
    assert rc == 0, adapter().ad_last_error()
    return Report(its.value, mv.value, hist[: hl.value].tolist(), bool(cv.value), st.value.decode(), x=x)
