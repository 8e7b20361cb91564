"""Python mirror of the reference chebmg interface, backed by the B200 library.

Names, argument meaning and error behaviour follow the reference C++ headers
(/root/reference/proj/include/chebmg): ``Domain``, ``StencilOperator``,
``build_problem``, ``ChebyshevConfig``, ``estimate_lambda_max``,
``chebyshev_smooth``, ``build_hierarchy``, ``CycleConfig`` /
``full_cycle`` / ``one_sided_cycle``, ``v_cycle``, ``preconditioner_apply``,
``SolveOptions``, ``SolveReport``, ``pcg``, ``pgmres``, ``CaseConfig``,
``run_case``.  ``std::invalid_argument`` maps to ``ValueError`` and
``std::out_of_range`` to ``IndexError``.

Vectors are ``torch.float64`` CUDA tensors (torch is the device-memory and
stream plumbing only); all arithmetic runs in libchebmg_b200.so.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Callable, List, Optional

import numpy as np
import torch

from . import _lib
from ._lib import check, lib


class Family(IntEnum):  # smoothers.hpp:14
    first = 0
    first_opt_lambda = 1
    fourth = 2
    fourth_opt = 3


def family_from_string(s: str) -> Family:
    try:
        return Family[s]
    except KeyError:
        raise ValueError(f"unknown smoother family: {s}") from None


def is_fourth_kind(f: Family) -> bool:
    return f in (Family.fourth, Family.fourth_opt)


# ---------------------------------------------------------------- context
class Context:
    """One CUDA device + the torch stream the library launches on."""

    _default: dict[int, "Context"] = {}

    def __init__(self, device: int = 0, stream: Optional[torch.cuda.Stream] = None):
        if not torch.cuda.is_available():
            raise RuntimeError("chebmg_b200 needs a CUDA device (no CPU fallback)")
        self.device = device
        s = stream if stream is not None else torch.cuda.current_stream(device)
        self.stream = s
        h = _lib.vp()
        check(lib.cmg_ctx_create(device, C.c_void_p(s.cuda_stream), C.byref(h)))
        self.h = h

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        if device not in cls._default:
            cls._default[device] = Context(device)
        return cls._default[device]

    def synchronize(self) -> None:
        check(lib.cmg_ctx_synchronize(self.h))

    def __del__(self):
        if getattr(self, "h", None) and self not in Context._default.values():
            try:
                lib.cmg_ctx_destroy(self.h)
            except Exception:  # interpreter shutdown
                pass
            self.h = None

    @staticmethod
    def kernel_launches() -> int:
        return int(lib.cmg_ctx_kernel_launches(None))

    def attach_nccl(self, unique_id: bytes, rank: int, nranks: int) -> None:
        buf = (C.c_ubyte * 128).from_buffer_copy(unique_id)
        check(lib.cmg_ctx_attach_nccl(self.h, buf, rank, nranks))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_ubyte * 128)()
        check(lib.cmg_nccl_unique_id(buf))
        return bytes(buf)


def _ptr(t: torch.Tensor) -> C.c_void_p:
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise ValueError("vectors must be contiguous float64 CUDA tensors")
    return C.c_void_p(t.data_ptr())


def _vec(n: int, ctx: Context) -> torch.Tensor:
    return torch.zeros(n, dtype=torch.float64, device=f"cuda:{ctx.device}")


# ---------------------------------------------------------------- core.hpp
def random_vector(n: int, seed: int) -> np.ndarray:
    """core.hpp:27-32 on the host (bit-identical mt19937_64 stream)."""
    out = np.empty(n, dtype=np.float64)
    check(lib.cmg_random_vector_host(n, seed, out.ctypes.data_as(_lib.dp)))
    return out


def dot(a: torch.Tensor, b: torch.Tensor, ctx: Optional[Context] = None) -> float:
    ctx = ctx or Context.default(a.device.index or 0)
    out = C.c_double()
    check(lib.cmg_dot(ctx.h, a.numel(), _ptr(a), _ptr(b), C.byref(out)))
    return out.value


def norm2(a: torch.Tensor, ctx: Optional[Context] = None) -> float:
    ctx = ctx or Context.default(a.device.index or 0)
    out = C.c_double()
    check(lib.cmg_norm2(ctx.h, a.numel(), _ptr(a), C.byref(out)))
    return out.value


# ---------------------------------------------------------------- domain / operators
@dataclass
class Domain:  # domain.hpp:12-26
    Lx: float = 1.0
    Ly: float = 1.0
    n: int = 0

    def __post_init__(self):
        if self.n < 2:
            raise ValueError("Domain: n must be at least 2")
        if self.Lx <= 0.0 or self.Ly <= 0.0:
            raise ValueError("Domain: side lengths must be positive")

    def interior_per_dim(self) -> int:
        return self.n - 1

    def unknowns(self) -> int:
        return (self.n - 1) ** 2

    def hx(self) -> float:
        return self.Lx / self.n

    def hy(self) -> float:
        return self.Ly / self.n


class DeviceOperator:
    """LinearOperatorLike over device vectors (operators.hpp:19-26)."""

    def __init__(self, handle, ctx: Context, owner=None):
        self.h = handle
        self.ctx = ctx
        self._owner = owner  # keeps the owning hierarchy alive

    def rows(self) -> int:
        return int(lib.cmg_op_rows(self.h))

    def cols(self) -> int:
        return self.rows()

    def vec_len(self) -> int:
        return int(lib.cmg_op_vec_len(self.h))

    def new_vector(self) -> torch.Tensor:
        return _vec(self.vec_len(), self.ctx)

    def apply(self, x: torch.Tensor, y: torch.Tensor) -> None:
        check(lib.cmg_op_apply(self.h, _ptr(x), _ptr(y)))

    def diagonal(self) -> torch.Tensor:
        d = self.new_vector()
        check(lib.cmg_op_diagonal(self.h, _ptr(d)))
        return d

    def applications(self) -> int:
        return int(lib.cmg_op_applications(self.h))

    def reset_applications(self) -> None:
        lib.cmg_op_reset_applications(self.h)


class StencilOperator(DeviceOperator):
    """Matrix-free 5-point Laplacian (operators.hpp:33-72)."""

    def __init__(self, dom: Domain, ctx: Optional[Context] = None):
        ctx = ctx or Context.default()
        h = _lib.vp()
        check(lib.cmg_fd_op_create(ctx.h, dom.n, dom.Lx, dom.Ly, C.byref(h)))
        super().__init__(h, ctx)
        self.domain = dom
        self._own = True

    def __del__(self):
        if getattr(self, "_own", False) and lib is not None:  # lib is None at interpreter shutdown
            lib.cmg_op_destroy(self.h)


@dataclass
class Problem:  # problem.hpp:20-25
    domain: Domain
    A: StencilOperator
    u_exact: torch.Tensor
    b: torch.Tensor


def build_problem_host(dom: Domain, rhs_seed: int) -> tuple[np.ndarray, np.ndarray]:
    m = dom.unknowns()
    u = np.empty(m)
    b = np.empty(m)
    check(lib.cmg_fd_build_problem_host(dom.n, dom.Lx, dom.Ly, rhs_seed, u.ctypes.data_as(_lib.dp),
                                        b.ctypes.data_as(_lib.dp)))
    return u, b


def build_problem(dom: Domain, rhs_seed: int, ctx: Optional[Context] = None) -> Problem:
    """problem.hpp:27-45: generated on the host (libm sin + mt19937_64), uploaded."""
    ctx = ctx or Context.default()
    u, b = build_problem_host(dom, rhs_seed)
    dev = f"cuda:{ctx.device}"
    return Problem(dom, StencilOperator(dom, ctx), torch.from_numpy(u).to(dev), torch.from_numpy(b).to(dev))


# ---------------------------------------------------------------- smoothers.hpp
@dataclass
class ChebyshevConfig:  # smoothers.hpp:41-57
    family: Family = Family.fourth
    order: int = 1
    lambda_tilde: float = 1.0
    lambda_max_multiplier: float = 1.03
    lambda_min_multiplier: float = 0.1

    def lambda_max(self) -> float:
        return self.lambda_max_multiplier * self.lambda_tilde

    def lambda_min(self) -> float:
        return self.lambda_min_multiplier * self.lambda_tilde

    def validate(self) -> None:
        if self.lambda_tilde <= 0.0:
            raise ValueError("ChebyshevConfig: lambda_tilde must be positive")
        if self.lambda_max() <= 0.0:
            raise ValueError("ChebyshevConfig: lambda_max must be positive")
        if not is_fourth_kind(self.family) and not (0.0 < self.lambda_min() < self.lambda_max()):
            raise ValueError("ChebyshevConfig: need 0 < lambda_min < lambda_max")

    def c(self) -> _lib.ChebConfig:
        return _lib.ChebConfig(int(self.family), self.lambda_tilde, self.lambda_max_multiplier,
                               self.lambda_min_multiplier)


BETA_MAX_ORDER = 20  # beta_table.hpp:83 (kBetaMaxOrder)


def beta_coefficients(k: int) -> list[float]:  # beta_table.hpp:86-92
    out = (C.c_double * max(k, 1))()
    check(lib.cmg_beta_coefficients(k, out))
    return list(out)[:k]


def jacobi_inverse_diagonal(diag: torch.Tensor, ctx: Optional[Context] = None) -> torch.Tensor:
    ctx = ctx or Context.default(diag.device.index or 0)
    inv = torch.empty_like(diag)
    check(lib.cmg_jacobi_inverse_diagonal(ctx.h, diag.numel(), _ptr(diag), _ptr(inv)))
    return inv


def estimate_lambda_max(A: DeviceOperator, inv_diag: torch.Tensor, iterations: int, seed: int) -> float:
    out = C.c_double()
    check(lib.cmg_estimate_lambda_max(A.h, _ptr(inv_diag), iterations, seed, C.byref(out)))
    return out.value


def chebyshev_smooth(A: DeviceOperator, inv_diag: torch.Tensor, cfg: ChebyshevConfig, order: int,
                     b: torch.Tensor, x: torch.Tensor, x_is_zero: bool) -> None:
    """smoothers.hpp:156-172 (one fused CUDA kernel per Chebyshev step)."""
    c = cfg.c()
    check(lib.cmg_chebyshev_smooth(A.h, _ptr(inv_diag), C.byref(c), order, _ptr(b), _ptr(x),
                                   1 if x_is_zero else 0))


# ---------------------------------------------------------------- multigrid.hpp
@dataclass
class CycleConfig:  # multigrid.hpp:53-57
    smoother: ChebyshevConfig = field(default_factory=ChebyshevConfig)
    k_pre: int = 1
    k_post: int = 1

    def c(self) -> _lib.CycleConfigC:
        return _lib.CycleConfigC(self.smoother.c(), self.k_pre, self.k_post)


def full_cycle(s: ChebyshevConfig, k: int) -> CycleConfig:
    return CycleConfig(s, k, k)


def one_sided_cycle(s: ChebyshevConfig, k: int) -> CycleConfig:
    return CycleConfig(s, 2 * k, 0)


class Hierarchy:
    """Two-level FD hierarchy (multigrid.hpp:21-48) resident on the GPU."""

    def __init__(self, dom: Domain, factor: int, eigen_iterations: int = 30, eigen_seed: int = 7,
                 ctx: Optional[Context] = None):
        self.ctx = ctx or Context.default()
        self.domain = dom
        self.factor = factor
        h = _lib.vp()
        check(lib.cmg_fd_hierarchy_create(self.ctx.h, dom.n, dom.Lx, dom.Ly, factor, eigen_iterations,
                                          eigen_seed, C.byref(h)))
        self.h = h
        self.A = DeviceOperator(lib.cmg_fd_hierarchy_op(h), self.ctx, owner=self)
        self.lambda_tilde = float(lib.cmg_fd_hierarchy_lambda_tilde(h))
        # Hierarchy::inv_diag (multigrid.hpp:24) -- same values the library holds
        self.inv_diag = jacobi_inverse_diagonal(self.A.diagonal(), self.ctx)

    def _clone_from(self, src: "Hierarchy", ctx: Context) -> None:
        """Same hierarchy on another context/stream (lambda_tilde copied)."""
        self.ctx = ctx
        self.domain = src.domain
        self.factor = src.factor
        h = _lib.vp()
        check(lib.cmg_fd_hierarchy_clone(src.h, ctx.h, C.byref(h)))
        self.h = h
        self.A = DeviceOperator(lib.cmg_fd_hierarchy_op(h), ctx, owner=self)
        self.lambda_tilde = float(lib.cmg_fd_hierarchy_lambda_tilde(h))
        self.inv_diag = jacobi_inverse_diagonal(self.A.diagonal(), ctx)

    def fine_dim(self) -> int:
        return self.A.rows()

    def coarse_dim(self) -> int:
        return int(lib.cmg_fd_hierarchy_coarse_dim(self.h))

    def prolong(self, xc: torch.Tensor) -> torch.Tensor:
        y = self.A.new_vector()
        check(lib.cmg_fd_prolong(self.h, _ptr(xc), _ptr(y)))
        return y

    def restrict(self, x: torch.Tensor) -> torch.Tensor:
        yc = _vec(self.coarse_dim(), self.ctx)
        check(lib.cmg_fd_restrict(self.h, _ptr(x), _ptr(yc)))
        return yc

    def coarse_solve(self, rc: torch.Tensor) -> torch.Tensor:
        ec = torch.empty_like(rc)
        check(lib.cmg_fd_coarse_solve(self.h, _ptr(rc), _ptr(ec)))
        return ec

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:  # lib is None at interpreter shutdown
            lib.cmg_fd_hierarchy_destroy(self.h)
            self.h = None


def build_hierarchy(dom: Domain, factor: int, eigen_iterations: int = 30, eigen_seed: int = 7,
                    ctx: Optional[Context] = None) -> Hierarchy:
    return Hierarchy(dom, factor, eigen_iterations, eigen_seed, ctx)


@dataclass
class CEstimate:
    """lanczos.hpp:39-44."""

    C: float = 0.0
    m: int = 0
    alpha: List[float] = field(default_factory=list)
    beta: List[float] = field(default_factory=list)


def estimate_C(h: Hierarchy, m: int = 20, seed: int = 99, reorthogonalize: bool = True) -> CEstimate:
    """Lanczos estimate of the approximation constant C (lanczos.hpp:97-155),
    run on the device (exact fine solve by fast diagonalisation)."""
    if m < 1:
        raise ValueError("estimate_C: need at least one iteration")
    a = (C.c_double * m)()
    b = (C.c_double * max(1, m - 1))()
    cval = C.c_double()
    steps = C.c_size_t()
    check(lib.cmg_fd_estimate_C(h.h, m, seed & (2**64 - 1), 1 if reorthogonalize else 0, C.byref(cval), a, b,
                                C.byref(steps)))
    k = steps.value
    return CEstimate(cval.value, m, list(a[:k]), list(b[: max(0, k - 1)]))


def v_cycle(h: Hierarchy, cfg: CycleConfig, b: torch.Tensor, x: torch.Tensor, x_is_zero: bool = False) -> None:
    c = cfg.c()
    check(lib.cmg_fd_v_cycle(h.h, C.byref(c), _ptr(b), _ptr(x), 1 if x_is_zero else 0))


def preconditioner_apply(h: Hierarchy, cfg: CycleConfig, v: torch.Tensor) -> torch.Tensor:
    z = torch.zeros_like(v)
    c = cfg.c()
    check(lib.cmg_fd_preconditioner_apply(h.h, C.byref(c), _ptr(v), _ptr(z)))
    return z


# ---------------------------------------------------------------- krylov.hpp
@dataclass
class SolveOptions:  # krylov.hpp:41-49
    tol: float = 1e-6
    maxit: int = 500
    restart: int = 30
    reorthogonalize: bool = True
    enforce_spd_preconditioner: bool = False

    def c(self) -> _lib.SolveOptionsC:
        return _lib.SolveOptionsC(self.tol, self.maxit, self.restart, int(self.reorthogonalize),
                                  int(self.enforce_spd_preconditioner))


@dataclass
class SolveReport:  # krylov.hpp:18-26
    iterations: int = 0
    fine_matvecs: int = 0
    residual_history: list = field(default_factory=list)
    rho: float = 1.0
    converged: bool = False
    status: str = ""
    wall_time_sec: float = 0.0


def convergence_rate(rep: SolveReport) -> float:  # krylov.hpp:30-37
    if not rep.residual_history or rep.iterations == 0:
        raise ValueError("convergence_rate: no iterations recorded")
    r0, rN = rep.residual_history[0], rep.residual_history[-1]
    if r0 == 0.0:
        raise ValueError("convergence_rate: zero initial residual")
    return math.exp(math.log(rN / r0) / rep.iterations)


class Preconditioner:
    """krylov.hpp:39 -- a native preconditioner handle."""

    def __init__(self, handle, keep=None):
        self.h = handle
        self._keep = keep

    def __call__(self, v: torch.Tensor) -> torch.Tensor:
        z = torch.zeros_like(v)
        check(lib.cmg_precond_apply(self.h, _ptr(v), _ptr(z)))
        return z

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:  # lib is None at interpreter shutdown
            lib.cmg_precond_destroy(self.h)
            self.h = None


def vcycle_preconditioner(h: Hierarchy, cfg: CycleConfig) -> Preconditioner:
    p = _lib.vp()
    c = cfg.c()
    check(lib.cmg_precond_fd_vcycle(h.h, C.byref(c), C.byref(p)))
    return Preconditioner(p, keep=h)


def identity_preconditioner(ctx: Optional[Context] = None) -> Preconditioner:
    ctx = ctx or Context.default()
    p = _lib.vp()
    check(lib.cmg_precond_identity(ctx.h, C.byref(p)))
    return Preconditioner(p)


def callback_preconditioner(fn: Callable[[torch.Tensor, torch.Tensor], None], n: int,
                            ctx: Optional[Context] = None) -> Preconditioner:
    """Wrap a Python callable fn(v, z) acting on device tensors of length n."""
    ctx = ctx or Context.default()
    dev = f"cuda:{ctx.device}"

    def tramp(user, vptr, zptr):
        v = _wrap_device(vptr, n, dev)
        z = _wrap_device(zptr, n, dev)
        fn(v, z)

    cb = _lib.PRECOND_FN(tramp)
    p = _lib.vp()
    check(lib.cmg_precond_callback(ctx.h, cb, None, C.byref(p)))
    return Preconditioner(p, keep=cb)


def _wrap_device(ptr: int, n: int, dev: str) -> torch.Tensor:
    # zero-copy view of a library-owned device buffer
    class _Cai:
        def __init__(self, p):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (p, False),
                                             "version": 3, "strides": None}

    return torch.as_tensor(_Cai(ptr), device=dev)


def _as_precond(M, A: DeviceOperator) -> Preconditioner:
    if isinstance(M, Preconditioner):
        return M
    if callable(M):
        def fn(v, z):
            z.copy_(M(v))
        return callback_preconditioner(fn, A.vec_len(), A.ctx)
    raise TypeError("M must be a Preconditioner or a callable")


def _report(r: _lib.SolveReportC, hist) -> SolveReport:
    n = min(r.history_len, len(hist))
    return SolveReport(int(r.iterations), int(r.fine_matvecs), list(hist[:n]), float(r.rho),
                       bool(r.converged), r.status.decode(), float(r.wall_time_sec))


def _solve(fn, A: DeviceOperator, M, b: torch.Tensor, x0: Optional[torch.Tensor], opts: SolveOptions):
    Mp = _as_precond(M, A)
    x = A.new_vector()
    hist = (C.c_double * (opts.maxit + 2))()
    rep = _lib.SolveReportC()
    rep.residual_history = C.cast(hist, _lib.dp)
    rep.history_capacity = opts.maxit + 2
    o = opts.c()
    check(fn(A.h, Mp.h, _ptr(b), _ptr(x0) if x0 is not None else None, _ptr(x), C.byref(o), C.byref(rep)))
    return x, _report(rep, hist)


def pcg(A: DeviceOperator, M, b: torch.Tensor, x0: Optional[torch.Tensor] = None,
        opts: Optional[SolveOptions] = None):
    """krylov.hpp:75-137 -> (x, SolveReport)."""
    return _solve(lib.cmg_pcg, A, M, b, x0, opts or SolveOptions())


def pgmres(A: DeviceOperator, M, b: torch.Tensor, x0: Optional[torch.Tensor] = None,
           opts: Optional[SolveOptions] = None):
    """krylov.hpp:144-264 -> (x, SolveReport)."""
    return _solve(lib.cmg_pgmres, A, M, b, x0, opts or SolveOptions())


def stationary_solve(A: DeviceOperator, M, b: torch.Tensor, tol: float, maxit: int) -> SolveReport:
    """harness.hpp:118-150."""
    Mp = _as_precond(M, A)
    x = A.new_vector()
    hist = (C.c_double * (maxit + 2))()
    rep = _lib.SolveReportC()
    rep.residual_history = C.cast(hist, _lib.dp)
    rep.history_capacity = maxit + 2
    check(lib.cmg_stationary_solve(A.h, Mp.h, _ptr(b), tol, maxit, _ptr(x), C.byref(rep)))
    return _report(rep, hist)


# ---------------------------------------------------------------- harness.hpp (the caller)
class Cycle(IntEnum):
    full = 0
    one_sided = 1


class Driver(IntEnum):
    pcg = 0
    pgmres = 1
    mg_solver = 2


def cycle_from_string(s: str) -> Cycle:  # harness.hpp:28-32
    try:
        return Cycle[s]
    except KeyError:
        raise ValueError(f"unknown cycle: {s}") from None


def driver_from_string(s: str) -> Driver:  # harness.hpp:36-41
    try:
        return Driver[s]
    except KeyError:
        raise ValueError(f"unknown driver: {s}") from None


def _fmt_g(v: float) -> str:
    """``std::ostream << double`` with the default stream flags (%g, precision 6)."""
    return f"{v:g}"


@dataclass
class Seeds:  # harness.hpp:52-56
    rhs: int = 1234
    eigen: int = 7
    tuning: int = 4321


@dataclass
class CaseConfig:  # harness.hpp:62-95
    Lx: float = 1.0
    n: int = 128
    factor: int = 2
    family: Family = Family.fourth
    k: int = 1
    cycle: Cycle = Cycle.one_sided
    driver: Driver = Driver.pcg
    tol: float = 1e-6
    restart: int = 30
    maxit: int = 500
    seeds: Seeds = field(default_factory=Seeds)
    lambda_max_multiplier: float = 1.03
    lambda_min_multiplier: float = 0.1
    eigen_iterations: int = 30
    estimate_c: bool = False

    def k_pre(self) -> int:
        return self.k if self.cycle == Cycle.full else 2 * self.k

    def k_post(self) -> int:
        return self.k if self.cycle == Cycle.full else 0

    def id(self) -> str:  # harness.hpp:82-87
        return (f"Lx{_fmt_g(self.Lx)}_f{self.factor}_{self.family.name}_k{self.k}_"
                f"{self.cycle.name}_{self.driver.name}")

    def validate(self) -> None:
        if self.k < 1:
            raise ValueError("CaseConfig: k must be >= 1")
        if self.factor < 2 or self.n % self.factor != 0:
            raise ValueError("CaseConfig: factor must divide n")
        if not self.tol > 0.0:
            raise ValueError("CaseConfig: tol must be positive")


@dataclass
class CaseResult:  # harness.hpp:97-104
    cfg: CaseConfig
    report: SolveReport
    lambda_tilde: float = 0.0
    C_est: Optional[float] = None
    tuned_lambda_min: Optional[float] = None
    note: str = ""
    x: Optional[torch.Tensor] = None


def default_tuning_candidates() -> list[float]:  # harness.hpp:170-176
    lo, hi = math.log(0.0125), math.log(0.4)
    return [math.exp(lo + (hi - lo) * i / 15.0) for i in range(16)]


def _smoother_config(cfg: CaseConfig, h: Hierarchy, lmin_mult: float) -> ChebyshevConfig:
    return ChebyshevConfig(cfg.family, 1, h.lambda_tilde, cfg.lambda_max_multiplier, lmin_mult)


def dispatch_driver(cfg: CaseConfig, h: Hierarchy, cc: CycleConfig, b: torch.Tensor):
    """harness.hpp:152-168 -> (x or None, SolveReport)."""
    M = vcycle_preconditioner(h, cc)
    opts = SolveOptions(tol=cfg.tol, maxit=cfg.maxit, restart=cfg.restart)
    if cfg.driver == Driver.pcg:
        return pcg(h.A, M, b, None, opts)
    if cfg.driver == Driver.pgmres:
        return pgmres(h.A, M, b, None, opts)
    return None, stationary_solve(h.A, M, b, cfg.tol, cfg.maxit)


@dataclass
class TuneRow:  # harness.hpp:178-181
    candidate: float
    report: SolveReport


def tune_lambda_min_table(cfg: CaseConfig, h: Hierarchy, candidates: list[float],
                          concurrent: bool = True) -> list[TuneRow]:
    """harness.hpp:186-201: one solve per lambda_min candidate against the
    seeded tuning right-hand side.  The candidate solves are independent, so
    with ``concurrent`` they run at the same time, each on its own CUDA stream
    with its own hierarchy scratch (the host threads sit in the library with
    the GIL released).  Reports are identical to the sequential run: every
    solve is deterministic and shares no mutable device state."""
    if not candidates:
        raise ValueError("tune_lambda_min_table: no candidates")
    dev = f"cuda:{h.ctx.device}"
    b_tune = torch.from_numpy(random_vector(h.fine_dim(), cfg.seeds.tuning)).to(dev)

    def one(cand: float, hh: Hierarchy) -> TuneRow:
        cc = CycleConfig(_smoother_config(cfg, hh, cand), cfg.k_pre(), cfg.k_post())
        return TuneRow(cand, dispatch_driver(cfg, hh, cc, b_tune)[1])

    if not concurrent or len(candidates) == 1:
        return [one(c, h) for c in candidates]
    import concurrent.futures as cf

    torch.cuda.synchronize(h.ctx.device)  # b_tune visible to every stream

    def worker(cand: float) -> TuneRow:
        stream = torch.cuda.Stream(h.ctx.device)
        with torch.cuda.stream(stream):  # torch-side allocations on the same stream
            ctx = Context(h.ctx.device, stream)
            hh = Hierarchy.__new__(Hierarchy)
            hh._clone_from(h, ctx)
            row = one(cand, hh)
            ctx.synchronize()
        return row

    with cf.ThreadPoolExecutor(max_workers=len(candidates)) as ex:
        return list(ex.map(worker, candidates))


def select_tuned(rows: list[TuneRow]) -> int:
    """harness.hpp:205-217: fewest iterations, ties by matvecs, first wins;
    len(rows) when nothing converged."""
    best = len(rows)
    for i, row in enumerate(rows):
        r = row.report
        if not r.converged:
            continue
        if best == len(rows) or r.iterations < rows[best].report.iterations or (
                r.iterations == rows[best].report.iterations and r.fine_matvecs < rows[best].report.fine_matvecs):
            best = i
    return best


def tune_lambda_min_empirical(cfg: CaseConfig, h: Hierarchy, candidates: list[float],
                              concurrent: bool = True) -> float:
    """harness.hpp:219-225."""
    rows = tune_lambda_min_table(cfg, h, candidates, concurrent)
    best = select_tuned(rows)
    if best == len(rows):
        raise RuntimeError(f"tune_lambda_min_empirical: all candidates failed for case {cfg.id()}")
    return rows[best].candidate


def run_case_with(cfg: CaseConfig, h: Hierarchy) -> CaseResult:
    """harness.hpp:230-251."""
    cfg.validate()
    res = CaseResult(cfg, SolveReport(), h.lambda_tilde)
    if cfg.cycle == Cycle.one_sided and cfg.driver == Driver.pcg:
        res.note = "pcg with an asymmetric one-sided preconditioner"
    lmin = cfg.lambda_min_multiplier
    if cfg.family == Family.first_opt_lambda:
        lmin = tune_lambda_min_empirical(cfg, h, default_tuning_candidates())
        res.tuned_lambda_min = lmin
    prob = build_problem(h.domain, cfg.seeds.rhs, h.ctx)
    cc = CycleConfig(_smoother_config(cfg, h, lmin), cfg.k_pre(), cfg.k_post())
    res.x, res.report = dispatch_driver(cfg, h, cc, prob.b)
    if cfg.estimate_c:
        res.C_est = estimate_C(h, 20, cfg.seeds.eigen).C
    return res


def run_case(cfg: CaseConfig, ctx: Optional[Context] = None) -> CaseResult:
    """harness.hpp:253-258."""
    cfg.validate()
    dom = Domain(cfg.Lx, 1.0, cfg.n)
    h = build_hierarchy(dom, cfg.factor, cfg.eigen_iterations, cfg.seeds.eigen, ctx)
    return run_case_with(cfg, h)


@dataclass
class SweepSpec:  # harness.hpp:262-269
    Lx: List[float] = field(default_factory=lambda: [1.0, 8.0, 64.0, 128.0])
    factors: List[int] = field(default_factory=lambda: [2, 16])
    families: List[Family] = field(default_factory=lambda: [Family.first, Family.fourth, Family.fourth_opt])
    ks: List[int] = field(default_factory=lambda: list(range(1, 11)))
    cycles: List[Cycle] = field(default_factory=lambda: [Cycle.full, Cycle.one_sided])
    base: CaseConfig = field(default_factory=CaseConfig)


@dataclass
class SweepResult:  # harness.hpp:271-276
    rows: List[CaseResult] = field(default_factory=list)
    best_per_group: dict = field(default_factory=dict)


def select_best_rows(sr: SweepResult) -> None:
    """harness.hpp:278-295: per (Lx, factor) the converged row with the fewest
    fine matvecs, ties by iterations, then smaller k, then row order."""
    sr.best_per_group = {}
    for i, r in enumerate(sr.rows):
        if not r.report.converged:
            continue
        key = (r.cfg.Lx, r.cfg.factor)
        cur = sr.best_per_group.get(key)
        if cur is None:
            sr.best_per_group[key] = i
            continue
        c = sr.rows[cur]
        if (r.report.fine_matvecs, r.report.iterations, r.cfg.k) < (c.report.fine_matvecs, c.report.iterations, c.cfg.k):
            sr.best_per_group[key] = i


def sweep_groups(spec: SweepSpec) -> list[tuple[float, int]]:
    return [(Lx, f) for Lx in spec.Lx for f in spec.factors]


def sweep_group_rows(spec: SweepSpec, Lx: float, factor: int, ctx: Optional[Context] = None) -> list[CaseResult]:
    """The rows of one (Lx, factor) group in reference order (harness.hpp:301-331);
    a row whose case throws becomes an error row."""
    import dataclasses

    probe = dataclasses.replace(spec.base, Lx=Lx, factor=factor)
    probe.validate()
    h = build_hierarchy(Domain(Lx, 1.0, probe.n), factor, probe.eigen_iterations, probe.seeds.eigen, ctx)
    C_shared = estimate_C(h, 20, probe.seeds.eigen).C if probe.estimate_c else None
    rows = []
    for fam in spec.families:
        for k in spec.ks:
            for cyc in spec.cycles:
                cfg = dataclasses.replace(probe, family=fam, k=k, cycle=cyc, estimate_c=False)
                try:
                    r = run_case_with(cfg, h)
                    r.x = None
                    r.C_est = C_shared
                except Exception as e:  # noqa: BLE001 -- the reference catches std::exception
                    r = CaseResult(cfg, SolveReport(residual_history=[0.0], status=f"error: {e}"), h.lambda_tilde)
                rows.append(r)
    return rows


def sweep(spec: SweepSpec, ctx: Optional[Context] = None, rank: int = 0, world: int = 1) -> SweepResult:
    """harness.hpp:297-337.  With world > 1 the (Lx, factor) groups are dealt
    round-robin to the ranks (one GPU each); every rank returns the rows of its
    groups and ``merge_sweep`` restores the reference row order."""
    out = SweepResult()
    for gi, (Lx, f) in enumerate(sweep_groups(spec)):
        if gi % world == rank:
            out.rows.extend(sweep_group_rows(spec, Lx, f, ctx))
    select_best_rows(out)
    return out


def merge_sweep(spec: SweepSpec, per_rank: list[SweepResult]) -> SweepResult:
    """Reassemble rank results (from ``sweep(..., rank, world)``) in reference row order."""
    world = len(per_rank)
    groups = sweep_groups(spec)
    queues = [list(p.rows) for p in per_rank]
    out = SweepResult()
    per_group = len(spec.families) * len(spec.ks) * len(spec.cycles)
    for gi, _ in enumerate(groups):
        q = queues[gi % world]
        out.rows.extend(q[:per_group])
        del q[:per_group]
    select_best_rows(out)
    return out
