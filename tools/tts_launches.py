#!/usr/bin/env python3
"""Launch list of ONE time-to-solution run (for ncu --profile-from-start off):

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
        --csv --log-file gpurun_out/tts_launches.csv python tools/tts_launches.py --case sem
    python tools/launch_summary.py gpurun_out/tts_launches.csv

--case sem : p-MG(7,3,1)-PGMRES(30), (8,0) 4th-kind half V-cycle, tol 1e-8 (bench.py's time_to_solution)
--case kras: paper Kershaw eps=0.05, E=36^3, 4th-opt Chebyshev-RAS (12,0), 4 PGMRES iterations
--case fd  : FD config 1, n=256 PGMRES + (4,0) 4th-kind half V-cycle, tol 1e-6 (bench.py's fd_config1)
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="sem", choices=["sem", "fd", "ras", "kras"])
    ap.add_argument("--E", type=int, default=64)
    args = ap.parse_args()
    import torch

    from paper_2210_03179_b200 import chebmg as cm
    from paper_2210_03179_b200 import sem

    ctx = cm.Context(0)
    if args.case == "kras":  # paper Kershaw eps=0.05 E=36^3, 4th-opt RAS(12,0), first 4 iterations
        P = sem.PMGHierarchy(sem.SemDesc(7, 36, 36, 36, geometry=sem.KERSHAW, eps=0.05), (7, 3, 1),
                             smoother=sem.RAS, ctx=ctx)
        A, b = P.A, P.A.rhs()
        M = P.preconditioner(cm.CycleConfig(cm.ChebyshevConfig(cm.Family.fourth_opt, 1, P.lambda_tilde[0]), 12, 0))
        opts = cm.SolveOptions(tol=1e-8, restart=30, maxit=4)
    elif args.case == "ras":  # configs[2]: Chebyshev-RAS (1,1), E=32^3
        P = sem.PMGHierarchy(sem.SemDesc(7, 32, 32, 32), (7, 3, 1), smoother=sem.RAS, ctx=ctx)
        A, b = P.A, P.A.rhs()
        M = P.preconditioner(cm.CycleConfig(cm.ChebyshevConfig(cm.Family.fourth, 1, P.lambda_tilde[0]), 1, 1))
        opts = cm.SolveOptions(tol=1e-8, restart=30, maxit=500)
    elif args.case == "sem":
        P = sem.PMGHierarchy(sem.SemDesc(7, args.E, args.E, args.E), (7, 3, 1), ctx=ctx)
        A, b = P.A, P.A.rhs()
        M = P.preconditioner(cm.CycleConfig(cm.ChebyshevConfig(cm.Family.fourth, 1, P.lambda_tilde[0]), 8, 0))
        opts = cm.SolveOptions(tol=1e-8, restart=30, maxit=500)
    else:
        h = cm.build_hierarchy(cm.Domain(1.0, 1.0, 256), 2, ctx=ctx)
        A, b = h.A, cm.build_problem(h.domain, 1234, ctx).b
        M = cm.vcycle_preconditioner(h, cm.CycleConfig(cm.ChebyshevConfig(cm.Family.fourth, 1, h.lambda_tilde), 4, 0))
        opts = cm.SolveOptions()
    cm.pgmres(A, M, b, None, opts)  # warm: workspace allocation
    torch.cuda.synchronize()
    l0 = cm.Context.kernel_launches()
    t0 = time.perf_counter()
    torch.cuda.profiler.start()
    _, rep = cm.pgmres(A, M, b, None, opts)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print({"case": args.case, "iterations": rep.iterations, "fine_matvecs": rep.fine_matvecs,
           "launches": cm.Context.kernel_launches() - l0, "wall_s": time.perf_counter() - t0})


if __name__ == "__main__":
    main()
