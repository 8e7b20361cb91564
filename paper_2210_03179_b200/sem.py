"""Spectral-element p-multigrid path (BASELINE.json north_star).

The reference library has no SEM code, so this layer extends the reference's
interface shapes to it: ``SemOperator`` is a LinearOperatorLike device
operator (operators.hpp:19-26) that the generic ``chebmg.chebyshev_smooth`` /
``chebmg.pcg`` / ``chebmg.pgmres`` drive unchanged; ``PMGHierarchy`` plays the
role of ``Hierarchy`` (multigrid.hpp:21-31) with the V-cycle of
multigrid.hpp:69-90 applied over the p-levels (e.g. 7 -> 3 -> 1).

Device vectors use the owned-slot layout (include/chebmg_b200.h);
``to_canonical`` / ``from_canonical`` convert to the lexicographic interior
ordering the oracle and the reference-template CPU baseline use.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import check, lib
from .chebmg import (ChebyshevConfig, Context, CycleConfig, DeviceOperator, Preconditioner, _ptr,
                     _wrap_device)

BOX, KERSHAW = 0, 1
JACOBI, ASM, RAS = 0, 1, 2


@dataclass
class SemDesc:
    order: int = 7
    ex: int = 4
    ey: int = 4
    ez: int = 4
    geometry: int = BOX
    eps: float = 1.0
    rank: int = 0
    nranks: int = 1

    def c(self) -> _lib.SemDesc:
        return _lib.SemDesc(self.order, self.ex, self.ey, self.ez, self.geometry, self.eps, self.rank, self.nranks)

    def with_order(self, order: int) -> "SemDesc":
        return SemDesc(order, self.ex, self.ey, self.ez, self.geometry, self.eps, self.rank, self.nranks)

    def unknowns(self) -> int:
        N = self.order
        return (N * self.ex - 1) * (N * self.ey - 1) * (N * self.ez - 1)

    def local_slots(self) -> int:
        d = self.c()
        return int(lib.cmg_sem_local_slots(C.byref(d)))

    def partition(self) -> tuple[int, int]:
        d = self.c()
        z0, z1 = C.c_int(), C.c_int()
        check(lib.cmg_sem_partition(C.byref(d), C.byref(z0), C.byref(z1)))
        return z0.value, z1.value


def slots_per_element(N: int) -> int:
    """csrc/sem_layout.hpp sem_nos: N^3 owned slots padded to an even count."""
    return (N * N * N + 1) & ~1


def slot_pos(N: int, a: int, b: int, c: int) -> int:
    """csrc/sem_layout.hpp sem_pos: interior-first element-local slot of owned node (a,b,c)."""
    if a < N - 1 and b < N - 1 and c < N - 1:
        return a + (N - 1) * (b + (N - 1) * c)
    base = (N - 1) ** 3
    if c == N - 1:
        return base + (N - 1) * (2 * N - 1) + b * N + a
    if b == N - 1:
        return base + c * (2 * N - 1) + (N - 1) + a
    return base + c * (2 * N - 1) + b


def slot_map(desc: SemDesc) -> np.ndarray:
    """Canonical interior index of every owned slot of this rank (-1 = padding)."""
    m = np.empty(desc.local_slots(), dtype=np.int64)
    d = desc.c()
    check(lib.cmg_sem_slot_map_host(C.byref(d), m.ctypes.data_as(C.POINTER(C.c_int64))))
    return m


def gs_map(desc: SemDesc) -> np.ndarray:
    """Gather-scatter map Q: canonical index of each local node of each local element (-1 Dirichlet)."""
    z0, z1 = desc.partition()
    E = desc.ex * desc.ey * (z1 - z0)
    m = np.empty(E * (desc.order + 1) ** 3, dtype=np.int64)
    d = desc.c()
    check(lib.cmg_sem_gs_map_host(C.byref(d), m.ctypes.data_as(C.POINTER(C.c_int64))))
    return m


class _Layout:
    def __init__(self, desc: SemDesc, ctx: Context):
        self.desc = desc
        self.ctx = ctx
        self.map = slot_map(desc)
        self.valid = self.map >= 0

    def to_canonical(self, v: torch.Tensor, out: Optional[np.ndarray] = None) -> np.ndarray:
        """Local slots -> this rank's entries of the canonical vector (others untouched/zero)."""
        h = v.detach().cpu().numpy()
        if out is None:
            out = np.zeros(self.desc.unknowns())
        out[self.map[self.valid]] = h[self.valid]
        return out

    def from_canonical(self, x: np.ndarray) -> torch.Tensor:
        h = np.zeros(self.map.size)
        h[self.valid] = x[self.map[self.valid]]
        return torch.from_numpy(h).to(f"cuda:{self.ctx.device}")


class SemOperator(DeviceOperator, _Layout):
    """A = Q^T A_L Q on one p-level (one rank's z-slab of elements)."""

    def __init__(self, desc: SemDesc, ctx: Optional[Context] = None, handle=None, owner=None):
        ctx = ctx or Context.default()
        own = handle is None
        if own:
            h = _lib.vp()
            d = desc.c()
            check(lib.cmg_sem_op_create(ctx.h, C.byref(d), C.byref(h)))
            handle = h
        DeviceOperator.__init__(self, handle, ctx, owner)
        _Layout.__init__(self, desc, ctx)
        self._own = own

    def rhs(self) -> torch.Tensor:
        """b = Q^T B f, f = 3 pi^2 sin(pi x) sin(pi y) sin(pi z)."""
        b = self.new_vector()
        check(lib.cmg_sem_rhs(self.h, _ptr(b)))
        return b

    def __del__(self):
        if getattr(self, "_own", False) and lib is not None:  # lib is None at interpreter shutdown
            lib.cmg_op_destroy(self.h)


class PMGHierarchy:
    """p-multigrid hierarchy resident on the GPU."""

    def __init__(self, desc: SemDesc, orders: Sequence[int] = (7, 3, 1), smoother: int = JACOBI,
                 eigen_iterations: int = 30, eigen_seed: int = 7, ctx: Optional[Context] = None):
        self.ctx = ctx or Context.default()
        self.desc = desc
        self.orders = list(orders)
        if desc.order != self.orders[0]:
            raise ValueError("pmg: orders[0] must equal the fine order")
        arr = (C.c_int * len(self.orders))(*self.orders)
        d = desc.c()
        h = _lib.vp()
        check(lib.cmg_pmg_create(self.ctx.h, C.byref(d), len(self.orders), arr, smoother, eigen_iterations,
                                 eigen_seed, C.byref(h)))
        self.h = h
        self.ops = [SemOperator(desc.with_order(o), self.ctx, handle=lib.cmg_pmg_op(h, l), owner=self)
                    for l, o in enumerate(self.orders)]
        self.lambda_tilde = [float(lib.cmg_pmg_lambda_tilde(h, l)) for l in range(len(self.orders))]

    @property
    def A(self) -> SemOperator:
        return self.ops[0]

    def inv_diag(self, level: int) -> torch.Tensor:
        op = self.ops[level]
        return _wrap_device(lib.cmg_pmg_inv_diag(self.h, level), op.vec_len(), f"cuda:{self.ctx.device}")

    def prolong(self, level: int, xc: torch.Tensor) -> torch.Tensor:
        y = self.ops[level].new_vector()
        check(lib.cmg_pmg_prolong(self.h, level, _ptr(xc), _ptr(y)))
        return y

    def restrict(self, level: int, xf: torch.Tensor) -> torch.Tensor:
        y = self.ops[level + 1].new_vector()
        check(lib.cmg_pmg_restrict(self.h, level, _ptr(xf), _ptr(y)))
        return y

    def coarse_solve(self, rc: torch.Tensor) -> torch.Tensor:
        e = self.ops[-1].new_vector()
        check(lib.cmg_pmg_coarse_solve(self.h, _ptr(rc), _ptr(e)))
        return e

    def smooth(self, level: int, cfg: ChebyshevConfig, order: int, b: torch.Tensor, x: torch.Tensor,
               x_is_zero: bool) -> None:
        c = cfg.c()
        check(lib.cmg_pmg_smooth(self.h, level, C.byref(c), order, _ptr(b), _ptr(x), int(x_is_zero)))

    def v_cycle(self, cfg: CycleConfig, b: torch.Tensor, x: torch.Tensor, x_is_zero: bool = False) -> None:
        c = cfg.c()
        check(lib.cmg_pmg_v_cycle(self.h, C.byref(c), _ptr(b), _ptr(x), int(x_is_zero)))

    def preconditioner_apply(self, cfg: CycleConfig, v: torch.Tensor) -> torch.Tensor:
        z = torch.zeros_like(v)
        self.v_cycle(cfg, v, z, True)
        return z

    def preconditioner(self, cfg: CycleConfig) -> Preconditioner:
        p = _lib.vp()
        c = cfg.c()
        check(lib.cmg_precond_pmg(self.h, C.byref(c), C.byref(p)))
        return Preconditioner(p, keep=self)

    def __del__(self):
        if getattr(self, "h", None) and lib is not None:  # lib is None at interpreter shutdown
            lib.cmg_pmg_destroy(self.h)
            self.h = None
