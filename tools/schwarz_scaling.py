#!/usr/bin/env python3
"""Chebyshev-Schwarz (ASM/RAS, FDM local solves) on the z-slab partition:
device time of one fine-level Chebyshev-Schwarz sweep and of the p-MG(7,3,1)
PGMRES(30) solve to 1e-8 (BASELINE configs[2] shape at E^3 elements), max over
ranks.  Rank 0 prints one JSON line.

    python tools/schwarz_scaling.py --E 64
    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/schwarz_scaling.py --E 64
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--E", type=int, default=64)
    ap.add_argument("--smoother", type=int, default=2, help="1 ASM, 2 RAS")
    ap.add_argument("--family", type=int, default=3, help="chebmg.Family (3 = optimised 4th kind)")
    ap.add_argument("--kpre", type=int, default=2)
    ap.add_argument("--kpost", type=int, default=0)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--eps", type=float, default=0.0, help="Kershaw deformation (0: undeformed box)")
    ap.add_argument("--ez", type=int, default=0, help="element layers (default E)")
    ap.add_argument("--lmin", type=float, default=0.1, help="lambda_min multiplier (1st kind)")
    args = ap.parse_args()
    import torch

    from paper_2210_03179_b200 import chebmg as cm
    from paper_2210_03179_b200 import sem

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    ctx = cm.Context(local)
    if world > 1:
        uid = [cm.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.attach_nccl(uid[0], rank, world)
    E = args.E
    geo = dict(geometry=sem.KERSHAW, eps=args.eps) if args.eps > 0 else {}
    d = sem.SemDesc(7, E, E, args.ez or E, rank=rank, nranks=world, **geo)
    P = sem.PMGHierarchy(d, (7, 3, 1), smoother=args.smoother, ctx=ctx)
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def max_ms(ms):
        if dist:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    b = P.A.rhs()
    # one fine-level Chebyshev-Schwarz sweep of order kpre (the (kpre,0) half cycle's smoother)
    ccfg = cm.ChebyshevConfig(cm.Family(args.family), args.kpre, P.lambda_tilde[0], lambda_min_multiplier=args.lmin)
    x = P.A.new_vector()
    for _ in range(3):
        P.smooth(0, ccfg, args.kpre, b, x, True)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.reps):
        P.smooth(0, ccfg, args.kpre, b, x, True)
    e1.record(stream)
    barrier()
    sweep_ms = max_ms(e0.elapsed_time(e1) / args.reps)

    cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family(args.family), 1, P.lambda_tilde[0],
                                            lambda_min_multiplier=args.lmin), args.kpre, args.kpost)
    M = P.preconditioner(cyc)
    opts = cm.SolveOptions(tol=1e-8, restart=30, maxit=500)
    cm.pgmres(P.A, M, b, None, opts)
    barrier()
    e0.record(stream)
    _, rep = cm.pgmres(P.A, M, b, None, opts)
    e1.record(stream)
    barrier()
    tts_ms = max_ms(e0.elapsed_time(e1))
    if rank == 0:
        print(json.dumps({"tool": "schwarz_scaling", "n_gpus": world, "E": E, "ez": args.ez or E, "N": 7,
                          "unknowns": d.unknowns(), "kershaw_eps": args.eps or None, "smoother": {1: "ASM", 2: "RAS"}[args.smoother],
                          "family": cm.Family(args.family).name, "cycle": f"({args.kpre},{args.kpost})", "lambda_min_multiplier": args.lmin,
                          "sweep_ms": sweep_ms, "iterations": rep.iterations, "fine_matvecs": rep.fine_matvecs,
                          "converged": rep.converged, "time_to_solution_s": tts_ms * 1e-3,
                          "ms_per_iteration": tts_ms / max(rep.iterations, 1)}), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
