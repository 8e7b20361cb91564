#!/usr/bin/env python3
"""Distributed FD parameter sweep (harness.hpp:297-337) -> sweep.csv (io.hpp:335-365).

The (Lx, factor) groups of the sweep are dealt round-robin to the ranks (one
GPU each, no data-path collective: every group builds its own hierarchy);
rank 0 gathers the rows, restores the reference row order and writes the same
16-column CSV the reference emits.

    python tools/sweep.py --config sweep.cfg --out DIR [--no-timing]
    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/sweep.py --config sweep.cfg --out DIR
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--no-timing", action="store_true")
    args = ap.parse_args()
    import torch

    from paper_2210_03179_b200 import chebmg as cm
    from paper_2210_03179_b200 import io as cio

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    spec = cio.sweep_spec_from_config(cio.Config.parse_file(args.config))
    ctx = cm.Context(local)
    t0 = time.perf_counter()
    part = cm.sweep(spec, ctx, rank, world)
    for r in part.rows:
        r.x = None
    elapsed = time.perf_counter() - t0
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")  # row objects only: host-side gather
        parts = [None] * world if rank == 0 else None
        dist.gather_object((part, elapsed), parts, dst=0)
        dist.destroy_process_group()
        if rank == 0:
            elapsed = max(p[1] for p in parts)
            sr = cm.merge_sweep(spec, [p[0] for p in parts])
    else:
        sr = part
    if rank == 0:
        os.makedirs(args.out, exist_ok=True)
        written = cio.emit_sweep(sr, args.out, opts=cio.CsvOptions(include_timing=not args.no_timing))
        best = {f"Lx{k[0]:g}_f{k[1]}": sr.rows[i].cfg.id() for k, i in sr.best_per_group.items()}
        print({"rows": len(sr.rows), "ranks": world, "seconds": round(elapsed, 3), "written": written, "best": best})


if __name__ == "__main__":
    main()
