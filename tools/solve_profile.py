"""One p-MG PGMRES solve (after a warm-up) between cudaProfilerStart/Stop, for
ncu --profile-from-start off launch lists of small configs:
    python tools/solve_profile.py --E 16 --kpre 8 --kpost 0 [--fd]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_03179_b200 import chebmg as cm, sem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--E", type=int, default=16)
ap.add_argument("--smoother", type=int, default=0)
ap.add_argument("--kpre", type=int, default=8)
ap.add_argument("--kpost", type=int, default=0)
a = ap.parse_args()
P = sem.PMGHierarchy(sem.SemDesc(7, a.E, a.E, a.E), (7, 3, 1), smoother=a.smoother)
cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family.fourth, 1, P.lambda_tilde[0]), a.kpre, a.kpost)
M = P.preconditioner(cyc)
b = P.A.rhs()
opts = cm.SolveOptions(tol=1e-8)
for _ in range(2):
    cm.pgmres(P.A, M, b, None, opts)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.profiler.start()
e0.record()
_, rep = cm.pgmres(P.A, M, b, None, opts)
e1.record()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("iterations", rep.iterations, "solve ms", e0.elapsed_time(e1))
