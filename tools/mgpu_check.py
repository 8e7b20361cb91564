#!/usr/bin/env python3
"""Element-partitioned SEM solve on WORLD_SIZE GPUs (one process per GPU).

Runs the p-MG(7,3,1)-preconditioned PGMRES on a z-slab partition and writes the
residual history, iteration counts and a solution checksum (as hex) to
--out (rank 0).  tests/test_multigpu.py runs it at 1 and 2/4 GPUs and checks
the histories are BITWISE identical (fixed-order QQ^T and layer reductions,
DESIGN.md §6) and that the NCCL halo path matches the single-GPU result.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/mgpu_check.py --out r2.json
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--E", type=int, default=4)
    ap.add_argument("--ez", type=int, default=8)
    ap.add_argument("--geometry", type=int, default=0)
    ap.add_argument("--out", required=True)
    ap.add_argument("--hash-only", action="store_true", help="write a sha256 of x instead of x itself")
    ap.add_argument("--kpre", type=int, default=4)
    ap.add_argument("--kpost", type=int, default=0)
    ap.add_argument("--family", type=int, default=2, help="0 first, 1 first_opt_lambda, 2 fourth, 3 fourth_opt")
    ap.add_argument("--smoother", type=int, default=0, help="0 Jacobi, 1 ASM, 2 RAS (Chebyshev-Schwarz)")
    args = ap.parse_args()
    import numpy as np
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
    d = sem.SemDesc(7, args.E, args.E, args.ez, geometry=args.geometry, eps=0.3, rank=rank, nranks=world)
    P = sem.PMGHierarchy(d, (7, 3, 1), smoother=args.smoother, ctx=ctx)
    b = P.A.rhs()
    cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family(args.family), 1, P.lambda_tilde[0]), args.kpre, args.kpost)
    x, rep = cm.pgmres(P.A, P.preconditioner(cyc), b, None, cm.SolveOptions(tol=1e-8))
    # gather the canonical solution on rank 0
    xc = P.A.to_canonical(x)
    if world > 1:
        t = torch.from_numpy(xc).cuda()
        dist.all_reduce(t)  # disjoint supports: sum == gather
        xc = t.cpu().numpy()
    if rank == 0:
        res = {"world": world, "iterations": rep.iterations, "fine_matvecs": rep.fine_matvecs,
               "history": [float(v).hex() for v in rep.residual_history],
               "lambda": [float(v).hex() for v in P.lambda_tilde],
               "x_norm": float(np.linalg.norm(xc)).hex(), "x_sum": float(np.sum(xc)).hex(),
               "x_sample": [float(v).hex() for v in xc[:: max(1, xc.size // 64)]]}
        if args.hash_only:
            import hashlib

            res["x_sha256"] = hashlib.sha256(np.ascontiguousarray(xc).tobytes()).hexdigest()
        with open(args.out, "w") as fh:
            json.dump(res, fh)
        if not args.hash_only:
            np.save(args.out + ".x.npy", xc)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
