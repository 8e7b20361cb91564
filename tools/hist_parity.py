"""Diagnostic: how close is the GPU SEM path to the reference-template CPU path?

Prints, per case, the iteration/matvec counts, the per-entry relative error of
the residual history, the error relative to h0, and the solution error; plus
bit-level agreement (max ulp distance) of the operator, diagonal and transfers.

    python tools/hist_parity.py [--E 16] [--quick]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_bind as ob  # noqa: E402
from paper_2210_03179_b200 import chebmg as cm, sem  # noqa: E402


def ulps(a, b):
    ai = np.ascontiguousarray(a).view(np.int64)
    bi = np.ascontiguousarray(b).view(np.int64)
    return int(np.max(np.abs(ai - bi))) if a.size else 0


def hist_stats(h, hr):
    h, hr = np.asarray(h), np.asarray(hr)
    n = min(h.size, hr.size)
    rel = np.abs(h[:n] - hr[:n]) / np.abs(hr[:n])
    return {"max_rel_entry": float(rel.max()), "max_abs_over_h0": float(np.max(np.abs(h[:n] - hr[:n])) / hr[0]),
            "worst_entry": int(rel.argmax()), "len": int(n)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--E", type=int, default=8)
    ap.add_argument("--geo", type=int, default=0)
    ap.add_argument("--eps", type=float, default=0.3)
    ap.add_argument("--cases", default="2:8:0,2:4:4,0:4:4,3:8:0")
    ap.add_argument("--smoother", type=int, default=0)
    a = ap.parse_args()
    E = a.E
    o = ob.OraclePmg((7, 3, 1), E, E, E, a.geo, a.eps, smoother=a.smoother, lib=ob.ref())
    P = sem.PMGHierarchy(sem.SemDesc(7, E, E, E, geometry=a.geo, eps=a.eps), (7, 3, 1), smoother=a.smoother)
    out = {"E": E, "geo": a.geo, "smoother": a.smoother,
           "lambda_rel": [abs(P.lambda_tilde[l] - o.lambda_tilde[l]) / o.lambda_tilde[l] for l in range(2)]}
    A = P.ops[0]
    x = ob.random_vector(o.n[0], 17)
    s0 = o.sem(0)
    out["apply_ulps"] = ulps(A.to_canonical(_apply(A, A.from_canonical(x))), s0.apply(x))
    out["diag_ulps"] = ulps(A.to_canonical(A.diagonal()), s0.diagonal())
    for l in (0, 1):
        xc = ob.random_vector(o.n[l + 1], 5)
        xf = ob.random_vector(o.n[l], 6)
        Pc, Pf = P.ops[l + 1], P.ops[l]
        out[f"prolong{l}_ulps"] = ulps(Pf.to_canonical(P.prolong(l, Pc.from_canonical(xc))), o.prolong(l, xc))
        out[f"restrict{l}_ulps"] = ulps(Pc.to_canonical(P.restrict(l, Pf.from_canonical(xf))), o.restrict(l, xf))
    print(json.dumps(out), flush=True)
    b = s0.rhs()
    for c in a.cases.split(","):
        fam, kpre, kpost = (int(t) for t in c.split(":"))
        oref = ob.ref_sem_solve(o, 1, fam, kpre, kpost, b, tol=1e-8)
        cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family(fam), 1, P.lambda_tilde[0]), kpre, kpost)
        xg, rep = cm.pgmres(P.A, P.preconditioner(cyc), P.A.from_canonical(b), None, cm.SolveOptions(tol=1e-8))
        xc = P.A.to_canonical(xg)
        r = {"case": c, "its": [rep.iterations, oref.iterations], "mv": [rep.fine_matvecs, oref.fine_matvecs],
             "x_rel": float(np.linalg.norm(xc - oref.x) / np.linalg.norm(oref.x))}
        r.update(hist_stats(rep.residual_history, oref.history))
        print(json.dumps(r), flush=True)


def _apply(A, x):
    y = A.new_vector()
    A.apply(x, y)
    return y


if __name__ == "__main__":
    main()
