"""Device time to solution of one BASELINE config (warm-up solve first), for A/B runs:
    python tools/tts_config.py --E 32 --smoother 2 --kpre 1 --kpost 1 [--geometry 1 --eps 0.3] [--reps 3]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--E", type=int, default=32)
ap.add_argument("--smoother", type=int, default=2)
ap.add_argument("--geometry", type=int, default=0)
ap.add_argument("--eps", type=float, default=1.0)
ap.add_argument("--family", type=int, default=2)
ap.add_argument("--kpre", type=int, default=1)
ap.add_argument("--kpost", type=int, default=1)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
import torch  # noqa: E402

from paper_2210_03179_b200 import chebmg as cm, sem  # noqa: E402

P = sem.PMGHierarchy(sem.SemDesc(7, a.E, a.E, a.E, geometry=a.geometry, eps=a.eps), (7, 3, 1), smoother=a.smoother)
cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family(a.family), 1, P.lambda_tilde[0]), a.kpre, a.kpost)
M = P.preconditioner(cyc)
b = P.A.rhs()
opts = cm.SolveOptions(tol=1e-8)
cm.pgmres(P.A, M, b, None, opts)
ts = []
for _ in range(a.reps):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, rep = cm.pgmres(P.A, M, b, None, opts)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(json.dumps({"E": a.E, "smoother": a.smoother, "cycle": [a.kpre, a.kpost], "iterations": rep.iterations,
                  "tts_ms": min(ts), "tts_all_ms": ts, "env": {k: v for k, v in os.environ.items() if k.startswith("CMG_")}}))
