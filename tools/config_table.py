#!/usr/bin/env python3
"""BASELINE configs[1..3] at full size on one GPU: iteration counts, fine
matvecs and time-to-solution of p-MG(7,3,1)-PGMRES(30) to 1e-8 for the cycle /
smoother / family grid each config names.  Writes a JSON table (--out).

  configs[1]  box N=7 E=16^3, full (k,k) vs half (2k,0), 1st / 4th / opt-4th kind Chebyshev-Jacobi
  configs[2]  box N=7 E=32^3, Chebyshev-ASM / -RAS (FDM local solves) vs Jacobi
  configs[3]  Kershaw-deformed box N=7 E=32^3, order-2k half vs order-k full V-cycle
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/config_table.json")
    ap.add_argument("--only", default="1,2,3")
    args = ap.parse_args()
    import torch

    from paper_2210_03179_b200 import chebmg as cm
    from paper_2210_03179_b200 import sem

    ctx = cm.Context(0)
    rows = []

    def run(tag, P, fam, kpre, kpost, lmin=0.1):
        cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family(fam), 1, P.lambda_tilde[0], lambda_min_multiplier=lmin),
                             kpre, kpost)
        M = P.preconditioner(cyc)
        b = P.A.rhs()
        opts = cm.SolveOptions(tol=1e-8, restart=30, maxit=500)
        cm.pgmres(P.A, M, b, None, opts)  # warm (workspace)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, rep = cm.pgmres(P.A, M, b, None, opts)
        e1.record()
        torch.cuda.synchronize()
        r = {"config": tag, "family": cm.Family(fam).name, "cycle": f"({kpre},{kpost})",
             "iterations": rep.iterations, "fine_matvecs": rep.fine_matvecs, "converged": rep.converged,
             "tts_ms": round(e0.elapsed_time(e1), 3), "rho": rep.rho, "lambda_min_multiplier": lmin}
        rows.append(r)
        print(json.dumps(r), flush=True)

    only = set(args.only.split(","))
    if "1" in only:
        P = sem.PMGHierarchy(sem.SemDesc(7, 16, 16, 16), (7, 3, 1), ctx=ctx)
        for fam in (0, 2, 3):
            for k in (1, 2, 4):
                run("configs[1] box E=16^3 Jacobi", P, fam, k, k)
                run("configs[1] box E=16^3 Jacobi", P, fam, 2 * k, 0)
        del P
    if "2" in only:
        for smoother, name in ((sem.ASM, "ASM"), (sem.RAS, "RAS"), (sem.JACOBI, "Jacobi")):
            P = sem.PMGHierarchy(sem.SemDesc(7, 32, 32, 32), (7, 3, 1), smoother=smoother, ctx=ctx)
            for fam in (2, 3):
                for kpre, kpost in ((1, 1), (2, 0), (2, 2), (4, 0)):
                    run(f"configs[2] box E=32^3 Chebyshev-{name}", P, fam, kpre, kpost)
            del P
    if "3" in only:
        for eps in (0.3, 0.1):
            P = sem.PMGHierarchy(sem.SemDesc(7, 32, 32, 32, geometry=sem.KERSHAW, eps=eps), (7, 3, 1), ctx=ctx)
            for fam in (2, 3):
                for k in (1, 2, 4):
                    run(f"configs[3] Kershaw eps={eps} E=32^3 Jacobi", P, fam, k, k)
                    run(f"configs[3] Kershaw eps={eps} E=32^3 Jacobi", P, fam, 2 * k, 0)
            del P
    if "paper" in only:
        # PAPER.md tab:ksp-comparison: Kershaw E=47K (36^3), p=7, 1st-kind Chebyshev-Jacobi (3,3),
        # (7,5,3,1) p-MG, PGMRES(30), tol 1e-8 -> 9 / 123 / 474 iterations at eps = 1 / 0.3 / 0.05
        # (the paper's coarsest level is one AMG V-cycle; here an exact p=1 solve)
        for eps, paper_its in ((1.0, 9), (0.3, 123), (0.05, 474)):
            P = sem.PMGHierarchy(sem.SemDesc(7, 36, 36, 36, geometry=sem.KERSHAW, eps=eps), (7, 5, 3, 1), ctx=ctx)
            run(f"paper Kershaw eps={eps} E=36^3 (7,5,3,1) [paper PGMRES: {paper_its} its]", P, 0, 3, 3)
            del P
    if "paper-ras" in only:
        # PAPER.md tab:fastest_solver_nekrs (:1016-1018, 6x V100): the fastest Chebyshev-RAS
        # configurations, (7,3,1) p-MG.  1st-kind with the empirically tuned lambda_min is
        # run here with the default lambda_min (family first).
        for eps, cases in ((1.0, ((0, 2, 2, "paper 1st lmin-opt RAS(2,2): 0.09 s, 8 its"), (3, 2, 2, ""))),
                           (0.3, ((0, 5, 5, "paper 1st lmin-opt RAS(5,5): 0.67 s, 28 its"), (3, 12, 0, ""))),
                           (0.05, ((3, 12, 0, "paper 4th-opt RAS(12,0): 2.40 s, 88 its"), (0, 5, 5, "")))):
            P = sem.PMGHierarchy(sem.SemDesc(7, 36, 36, 36, geometry=sem.KERSHAW, eps=eps), (7, 3, 1),
                                 smoother=sem.RAS, ctx=ctx)
            for fam, kpre, kpost, note in cases:
                run(f"paper Kershaw eps={eps} E=36^3 (7,3,1) RAS" + (f" [{note}]" if note else ""), P, fam, kpre,
                    kpost)
            del P
    if "paper-ras-tune" in only:
        # the paper's 1st-kind rows use an empirically tuned lambda_min:
        # scan the multiplier like harness.hpp:172-225 does for the FD problem
        for eps, k in ((1.0, 2), (0.3, 5)):
            P = sem.PMGHierarchy(sem.SemDesc(7, 36, 36, 36, geometry=sem.KERSHAW, eps=eps), (7, 3, 1),
                                 smoother=sem.RAS, ctx=ctx)
            for lmin in (0.02, 0.05, 0.1, 0.2, 0.3, 0.4, 0.5, 0.6):
                run(f"paper Kershaw eps={eps} E=36^3 (7,3,1) RAS 1st kind lambda_min scan", P, 0, k, k, lmin)
            del P
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump({"device": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%d %H:%M:%S"),
                   "rows": rows}, fh, indent=1)


if __name__ == "__main__":
    main()
