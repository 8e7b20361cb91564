"""Setup + warm sweeps + ONE profiled 4th-kind order-8 Chebyshev-Jacobi sweep at
N=7, E^3 (the bench step), bracketed by cudaProfilerStart/Stop, for
`ncu --profile-from-start off` captures (tools/prof_r02.sh)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_03179_b200 import chebmg as cm, sem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--E", type=int, default=64)
ap.add_argument("--order", type=int, default=8)
ap.add_argument("--solve", action="store_true", help="profile one p-MG PGMRES solve instead of a sweep")
a = ap.parse_args()
P = sem.PMGHierarchy(sem.SemDesc(7, a.E, a.E, a.E), (7, 3, 1))
A = P.A
invd = P.inv_diag(0)
b = A.rhs()
x = A.new_vector()
x.copy_(torch.rand_like(x) * torch.from_numpy(A.valid.astype(np.float64)).to(x.device))
cfg = cm.ChebyshevConfig(cm.Family.fourth, a.order, P.lambda_tilde[0])
cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family.fourth, 1, P.lambda_tilde[0]), 8, 0)
M = P.preconditioner(cyc)


def work():
    if a.solve:
        cm.pgmres(A, M, b, None, cm.SolveOptions(tol=1e-8))
    else:
        cm.chebyshev_smooth(A, invd, cfg, a.order, b, x, False)


for _ in range(2):
    work()
torch.cuda.synchronize()
torch.cuda.profiler.start()
work()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
