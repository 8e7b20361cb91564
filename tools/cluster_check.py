"""Hashes of A x, one 4th-kind order-8 sweep and a short p-MG PGMRES solve on a
few box and Kershaw meshes, for comparing library variants or knobs bit for bit
(used for the 2x2x2-cluster K1 experiment, profiles/r02/ab_k1_cluster.txt):
    CMG_LIB=... python tools/cluster_check.py   (one line per case)."""
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_03179_b200 import chebmg as cm, sem  # noqa: E402


def h(t):
    return hashlib.sha256(t.detach().cpu().numpy().tobytes()).hexdigest()[:16]


for (E, geo, eps) in [((4, 4, 4), 0, 1.0), ((8, 6, 4), 1, 0.3), ((16, 16, 16), 0, 1.0), ((6, 8, 10), 1, 0.3)]:
    P = sem.PMGHierarchy(sem.SemDesc(7, *E, geometry=geo, eps=eps), (7, 3, 1))
    A = P.A
    g = torch.Generator(device="cpu").manual_seed(5)
    valid = torch.from_numpy(A.valid.astype(np.float64)).to(A.new_vector().device)
    x = (torch.rand(A.new_vector().shape, generator=g, dtype=torch.float64).to(valid.device) - 0.5) * valid
    y = A.new_vector()
    A.apply(x, y)
    b = A.rhs()
    xs = x.clone()
    cm.chebyshev_smooth(A, P.inv_diag(0), cm.ChebyshevConfig(cm.Family.fourth, 8, P.lambda_tilde[0]), 8, b, xs, False)
    cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family.fourth, 1, P.lambda_tilde[0]), 8, 0)
    xsol, rep = cm.pgmres(A, P.preconditioner(cyc), b, None, cm.SolveOptions(tol=1e-8, maxit=50, restart=30))
    print(E, geo, "Ax", h(y), "sweep", h(xs), "solve", h(xsol), rep.iterations, f"{rep.residual_history[-1]:.6e}",
          flush=True)
    del P
