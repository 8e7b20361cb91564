#!/usr/bin/env python3
"""bench.py -- BASELINE.json metric on B200.

Metric: "GDOF/s per Chebyshev smoother sweep; p-MG-GMRES time-to-solution".
A *step* is one 4th-kind Chebyshev-Jacobi smoother sweep of order 8 (the
(2k,0) half-V-cycle smoother with k=4) on the fine level of the SEM Poisson
problem N=7, E=64^3 (BASELINE north-star target; configs[4] is the same
problem element-partitioned over 2/4/8 GPUs).  Each step = 8 fused
Ax+QQ^T+Chebyshev passes (warm start: the residual pass plus 7 steps).
`value` = total unknowns x 8 x K / (max over ranks of the device time) in
GDOF-step/s.  Extra keys carry the full p-MG(7,3,1)-PGMRES time-to-solution,
the FD config-1 solve, the roofline and the CPU baseline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


# ---------------------------------------------------------------- clocks sampler
class Clocks:
    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _nvml_handle(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            try:
                import torch

                p = torch.cuda.get_device_properties(self.device)
                bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
                return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.device)
        except Exception:
            return None, None

    def _run(self):
        nv, h = self._nvml_handle()
        if h is not None:  # NVML: a sample every 5 ms inside the timed region
            bits = [("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
                    ("sw_power_cap", 0x4)]
            try:
                mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                while not self._stop.is_set():
                    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append([str(sm), str(mx), ""] + ["Active" if r & b else "Not Active" for _, b in bits])
                    self._stop.wait(0.005)
                return
            except Exception:
                self.samples = []
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.samples:  # region shorter than one poll: one sample at its end
            self._stop.clear()
            t = threading.Thread(target=self._run, daemon=True)
            t.start()
            time.sleep(0.05)
            self._stop.set()
            t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max((float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and
                          s[3 + i].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------- CPU reference arm
def measured_traffic(E, order, world):
    """DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of the K1/K2 launches of
    one sweep from the committed ncu --set full capture (tools/ncu_traffic.py ->
    profiles/r02/sem_sweep_traffic.json), scaled per element to this run's slab."""
    path = os.path.join(ROOT, "profiles", "r02", "sem_sweep_traffic.json")
    try:
        with open(path) as fh:
            t = json.load(fh)
    except Exception:
        return None
    scale = (E ** 3 / world) / t["elements"]
    return {"traffic": t["dram_bytes_per_sweep"] * scale * order / t["order"],
            "traffic_source": f"ncu --set full, {t['source']}", "traffic_over_algorithmic": t["ratio"]}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def replica_bytes(E: int) -> float:
    """Host memory of one reference sweep context at E^3 (oracle_sem.c level:
    G, mass, coordinates, gather map = 88 B per local node; b, x, inv_diag and
    smooth_fourth's r, d, t + slack = 7 vectors)."""
    n = (7 * E - 1) ** 3
    return 88.0 * 512 * E ** 3 + 7 * 8.0 * n


def _sweep_replica(E, order, barrier, q):
    """One reference chebyshev_smooth sweep (oracle/_ref: the reference template over
    the SEM restatement, single thread) at full size, after every replica's setup."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import ctypes as C

    import oracle_bind as ob

    L = ob.ref()
    L.ref_sem_bench_create.restype = C.c_void_p
    L.ref_sem_bench_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, ob.sz, C.c_uint64]
    L.ref_sem_bench_n.restype = ob.sz
    L.ref_sem_bench_n.argtypes = [C.c_void_p]
    L.ref_sem_bench_sweep.argtypes = [C.c_void_p, C.c_int, ob.sz]
    L.ref_sem_bench_destroy.argtypes = [C.c_void_p]
    t0 = time.perf_counter()
    h = L.ref_sem_bench_create(7, E, 0, 1.0, 3, 7)
    setup = time.perf_counter() - t0
    n = L.ref_sem_bench_n(h) if h else 0
    if barrier is not None:
        barrier.wait()
    t1 = time.perf_counter()
    rc = L.ref_sem_bench_sweep(h, 2, order) if h else -1
    dt = time.perf_counter() - t1
    L.ref_sem_bench_destroy(h)
    q.put((n, dt, setup, rc))


def cpu_reference_sweeps(E: int, order: int, replicas: int):
    """`replicas` concurrent single-thread reference sweeps at E^3 (one each)."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    bar = ctx.Barrier(replicas) if replicas > 1 else None
    ps = [ctx.Process(target=_sweep_replica, args=(E, order, bar, q)) for _ in range(replicas)]
    for p in ps:
        p.start()
    outs = [q.get() for _ in ps]
    for p in ps:
        p.join()
    if any(o[3] != 0 for o in outs):
        raise RuntimeError("reference sweep failed")
    n = outs[0][0]
    value = sum(n * order / o[1] for o in outs) / 1e9
    sample = (f"{replicas} concurrent single-thread replicas x 1 sweep: SEM N=7 E={E}^3 ({n} unknowns) 4th-kind "
              f"Chebyshev-Jacobi order {order}, reference chebyshev_smooth template (oracle/_ref) over the "
              f"restated SEM operator; sweep {min(o[1] for o in outs):.1f}-{max(o[1] for o in outs):.1f} s, "
              f"setup {max(o[2] for o in outs):.0f} s (untimed); CPU: {cpu_model()}")
    return value, "reference", sample


def reference_replicas(E: int) -> int:
    """All host cores, capped by available host memory (~17 GB per E=64^3 replica)."""
    cores = os.cpu_count() or 1
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = 16e9
    return max(1, min(cores, int(0.6 * avail / replica_bytes(E))))


def run_reference_arm(args):
    """--impl reference: the reference CPU path on the host cores, same config as
    the GPU arm (N=7, E^3 = --E), one order-8 sweep per replica (the bounded
    sample; the reference is single-threaded by contract, core.hpp:34-35, so the
    cores run independent replicas).  K/W do not apply: one E=64^3 sweep is ~40 s
    of single-core work."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    E = args.cpu_E or args.E
    P = reference_replicas(E)
    t0 = time.perf_counter()
    value, kind, sample = cpu_reference_sweeps(E, args.order, P)
    wall = time.perf_counter() - t0
    n = (7 * E - 1) ** 3
    line = {
        "impl": "reference", "metric": "GDOF/s per Chebyshev smoother sweep", "value": value,
        "unit": "GDOF-step/s", "n_gpus": args.gpus, "steps": 1, "warmup": 0,
        "ms_per_step": n * args.order / (value * 1e9) * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(E, args.order, n, 1),
        "cpu_baseline": {"value": value, "unit": "GDOF-step/s", "cores": P, "kind": kind, "sample": sample,
                         "cpu": cpu_model(), "host_cores": os.cpu_count()},
        "e2e": {"value": value, "unit": "GDOF-step/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)


def sweep_bytes(E, order, n_glob):
    """Algorithmic DRAM bytes of one warm sweep: 48 B per local node on
    every pass; per unknown 40 B (init pass), 64 B (middle steps), 48 B (fused last step)."""
    return order * 48 * 512 * E ** 3 + (40 + 64 * (order - 2) + 48) * n_glob


def config_of(E, order, n_glob, world):
    """The workload -- identical for the GPU arm at any N and the reference arm
    (the partition is reported next to it, not in it)."""
    return {"workload": f"SEM Poisson box [-1/2,1/2]^3 N=7 E={E}^3 ({n_glob} unknowns), 4th-kind "
                        f"Chebyshev-Jacobi sweep order {order} on the fine level of p-MG(7,3,1), warm start",
            "N": 7, "E": E ** 3, "unknowns": n_glob,
            "l2": f"inputs larger than L2 (each vector {n_glob * 8 / 1e6:.0f} MB, geometric factors "
                  f"{6 * 512 * E ** 3 * 8 / 1e9:.1f} GB in total)"}


def fd_reference_run_case():
    """FD config 1 through the reference's own harness (oracle/_ref run_case_with,
    harness.hpp:230-258): n=256, factor 2, 4th kind, one-sided k=2 ((4,0)), PGMRES,
    tol 1e-6; hierarchy built untimed, as on the GPU side."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_bind as ob

    h = ob.RefHierarchy(256, 1.0, 2)
    best, wall, rep = None, [], None
    for _ in range(5):
        t0 = time.perf_counter()
        rep = h.run_case(2, 2, 1, 1)
        wall.append(time.perf_counter() - t0)
    return {"kind": "reference", "run_case_ms": min(wall) * 1e3, "pgmres_ms": rep.wall_time_sec * 1e3,
            "iterations": rep.iterations, "fine_matvecs": rep.fine_matvecs, "cores": 1, "cpu": cpu_model(),
            "sample": "reference run_case_with (build_problem + pgmres) on one core, best of 5"}


# ---------------------------------------------------------------- BASELINE configs[1..3]
def baseline_config_solves(cm, sem, ctx, stream):
    """Full-size solves of the other BASELINE configs on this GPU (p-MG(7,3,1)
    PGMRES(30), tol 1e-8): iterations, fine matvecs and device time to
    solution, each after a warm-up solve.  tools/config_table.py has the full grid."""
    import torch

    def solve(P, fam, kpre, kpost):
        cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family(fam), 1, P.lambda_tilde[0]), kpre, kpost)
        M = P.preconditioner(cyc)
        b = P.A.rhs()
        opts = cm.SolveOptions(tol=1e-8, restart=30, maxit=500)
        cm.pgmres(P.A, M, b, None, opts)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, rep = cm.pgmres(P.A, M, b, None, opts)
        e1.record(stream)
        torch.cuda.synchronize()
        return {"cycle": f"({kpre},{kpost})", "family": cm.Family(fam).name, "iterations": rep.iterations,
                "fine_matvecs": rep.fine_matvecs, "converged": rep.converged,
                "time_to_solution_ms": e0.elapsed_time(e1)}

    out = {}
    P = sem.PMGHierarchy(sem.SemDesc(7, 16, 16, 16), (7, 3, 1), ctx=ctx)
    out["configs[1] box N=7 E=16^3, Chebyshev-Jacobi"] = [solve(P, f, kp, kq) for f in (0, 2, 3)
                                                          for kp, kq in ((8, 0), (4, 4))]
    del P
    rows = []
    for smoother, name in ((sem.RAS, "RAS"), (sem.ASM, "ASM")):
        P = sem.PMGHierarchy(sem.SemDesc(7, 32, 32, 32), (7, 3, 1), smoother=smoother, ctx=ctx)
        rows += [dict(solve(P, 2, kp, kq), smoother=name) for kp, kq in ((2, 0), (1, 1))]
        del P
    out["configs[2] box N=7 E=32^3, Chebyshev-Schwarz (FDM local solves)"] = rows
    P = sem.PMGHierarchy(sem.SemDesc(7, 32, 32, 32, geometry=sem.KERSHAW, eps=0.3), (7, 3, 1), ctx=ctx)
    out["configs[3] Kershaw eps=0.3 N=7 E=32^3, Chebyshev-Jacobi"] = [solve(P, 2, kp, kq)
                                                                     for kp, kq in ((8, 0), (4, 4))]
    del P
    return out


# ---------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--E", type=int, default=64, help="elements per direction (N=7)")
    ap.add_argument("--order", type=int, default=8)
    ap.add_argument("--cpu-E", dest="cpu_E", type=int, default=0, help="CPU legs' E (default: --E)")
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the BASELINE configs[1..3] solves")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
        return

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

    E, order = args.E, args.order
    desc = sem.SemDesc(7, E, E, E, rank=rank, nranks=world)
    t_setup = time.perf_counter()
    P = sem.PMGHierarchy(desc, (7, 3, 1), ctx=ctx)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    A = P.A
    invd = P.inv_diag(0)
    n_glob = desc.unknowns()
    b = A.rhs()
    x = A.new_vector()
    x.copy_(torch.rand_like(x) * torch.from_numpy(A.valid.astype(np.float64)).to(x.device))
    cfg = cm.ChebyshevConfig(cm.Family.fourth, order, P.lambda_tilde[0])
    stream = torch.cuda.current_stream()

    def sweep():
        cm.chebyshev_smooth(A, invd, cfg, order, b, x, False)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        sweep()
    barrier()
    l0 = cm.Context.kernel_launches()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with Clocks(local) as clk:
        ev[0].record(stream)
        for k in range(args.steps):
            sweep()
            ev[k + 1].record(stream)
        barrier()
    launches = cm.Context.kernel_launches() - l0
    step_ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
    t_ms = ev[0].elapsed_time(ev[-1])
    if dist:
        tt = torch.tensor([t_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    ms_per_step = t_ms / args.steps
    value = n_glob * order * args.steps / (t_ms * 1e-3) / 1e9

    # roofline of the fused sweep (K1 + K2 per pass), SURVEY §8(d) algorithmic bytes
    # per pass: 48 B per local node (6 geometric factors) plus, per global unknown,
    # 40 B on the residual-initialising pass (gather x; read b, invD; write r, d),
    # 64 B on a middle step (gather d; read d, x, r, invD; write x, r, d') and 48 B
    # on the fused last step (no r, d writes): 8*48 N_L + (40 + 6*64 + 48) N_G at order 8
    per_gpu_bytes = sweep_bytes(E, order, n_glob) / world
    peak, peak_src = peaks()
    achieved = per_gpu_bytes / (ms_per_step * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": None, "kernel": "fused Chebyshev-Jacobi sweep (sem K1 element kernel + K2 shared-node "
                                       "kernel, 8 passes)",
            "algorithmic_bytes_per_sweep": per_gpu_bytes, "peak_source": peak_src}
    tr = measured_traffic(E, order, world)
    if tr:
        roof.update(tr)

    # e2e through the C ABI with host buffers, as a host caller of the library
    # sees it: every step cmg_upload(b), cmg_upload(x) from
    # pinned host memory, cmg_chebyshev_smooth, cmg_download(x) -- each copy
    # synchronous on the context's stream, timed with CUDA events on that stream
    from paper_2210_03179_b200 import _lib

    hb = b.detach().cpu().pin_memory()
    hx = x.detach().cpu().pin_memory()
    hout = torch.empty_like(hx).pin_memory()
    db, dxv = torch.empty_like(b), torch.empty_like(x)
    nbytes = b.numel() * 8
    cc = cfg.c()

    def abi_step():
        _lib.check(_lib.lib.cmg_upload(ctx.h, C.c_void_p(db.data_ptr()), C.c_void_p(hb.data_ptr()), nbytes))
        _lib.check(_lib.lib.cmg_upload(ctx.h, C.c_void_p(dxv.data_ptr()), C.c_void_p(hx.data_ptr()), nbytes))
        _lib.check(_lib.lib.cmg_chebyshev_smooth(A.h, C.c_void_p(invd.data_ptr()), C.byref(cc), order,
                                                 C.c_void_p(db.data_ptr()), C.c_void_p(dxv.data_ptr()), 0))
        _lib.check(_lib.lib.cmg_download(ctx.h, C.c_void_p(hout.data_ptr()), C.c_void_p(dxv.data_ptr()), nbytes))

    abi_step()
    barrier()
    e2e_steps = max(3, min(args.steps, 8))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        abi_step()
    e1.record(stream)
    barrier()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    if dist:
        tt = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e = {"value": n_glob * order / (e2e_ms * 1e-3) / 1e9, "unit": "GDOF-step/s",
           "h2d_bytes_per_step": 2 * nbytes * world, "d2h_bytes_per_step": nbytes * world, "ms_per_step": e2e_ms,
           "path": "C ABI cmg_upload x2 + cmg_chebyshev_smooth + cmg_download per step, pinned host buffers"}

    # the same host-buffer workload pipelined the way a solver service would run it:
    # step i+1's inputs stream in on a copy stream while step i computes and step
    # i-1's result streams out on a second one (triple-buffered)
    NB = 3
    bufs = [(b, x)] + [(torch.empty_like(b), torch.empty_like(x)) for _ in range(NB - 1)]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(NB)]
    ev_done = [torch.cuda.Event() for _ in range(NB)]
    ev_free = [torch.cuda.Event() for _ in range(NB)]
    barrier()
    e0.record(stream)
    s_in.wait_event(e0)
    for i in range(e2e_steps):
        k = i % NB
        bb, xx = bufs[k]
        with torch.cuda.stream(s_in):
            if i >= NB:
                s_in.wait_event(ev_free[k])  # the D2H of step i-NB has read this x
            bb.copy_(hb, non_blocking=True)
            xx.copy_(hx, non_blocking=True)
            ev_in[k].record(s_in)
        stream.wait_event(ev_in[k])
        cm.chebyshev_smooth(A, invd, cfg, order, bb, xx, False)
        ev_done[k].record(stream)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_done[k])
            hout.copy_(xx, non_blocking=True)
            ev_free[k].record(s_out)
    stream.wait_event(ev_free[(e2e_steps - 1) % NB])
    e1.record(stream)
    barrier()
    pipe_ms = e0.elapsed_time(e1) / e2e_steps
    if dist:
        tt = torch.tensor([pipe_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        pipe_ms = float(tt.item())
    e2e_pipe = {"value": n_glob * order / (pipe_ms * 1e-3) / 1e9, "unit": "GDOF-step/s", "ms_per_step": pipe_ms,
                "path": "torch pinned copies on two copy streams around cmg_chebyshev_smooth, triple-buffered"}
    del bufs

    # p-MG(7,3,1)-PGMRES time to solution (tol 1e-8, restart 30), half V-cycle (8,0)
    tts = None
    if not args.no_solve:
        cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family.fourth, 1, P.lambda_tilde[0]), 8, 0)
        M = P.preconditioner(cyc)
        # warm-up solve: allocates the PGMRES(30) workspace (V, Z: 61 vectors) once
        cm.pgmres(A, M, b, None, cm.SolveOptions(tol=1e-8, restart=30, maxit=500))
        barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        xs, rep = cm.pgmres(A, M, b, None, cm.SolveOptions(tol=1e-8, restart=30, maxit=500))
        s1.record(stream)
        barrier()
        sms = s0.elapsed_time(s1)
        if dist:
            tt = torch.tensor([sms], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            sms = float(tt.item())
        tts = {"solver": "PGMRES(30) + p-MG(7,3,1) 4th-kind Chebyshev-Jacobi half V-cycle (8,0)", "tol": 1e-8,
               "iterations": rep.iterations, "fine_matvecs": rep.fine_matvecs, "converged": rep.converged,
               "time_to_solution_s": sms * 1e-3, "ms_per_iteration": sms / max(rep.iterations, 1),
               "final_rel_residual": rep.residual_history[-1] / rep.residual_history[0]}

    fd = None
    cpu = None
    configs = None
    if rank == 0 and world == 1:
        # FD config 1: n=256 (255^2 unknowns), PGMRES + 4th-kind (4,0) half V-cycle, factor 2, Lx=1
        h = cm.build_hierarchy(cm.Domain(1.0, 1.0, 256), 2, ctx=ctx)
        prob = cm.build_problem(h.domain, 1234, ctx)
        Mfd = cm.vcycle_preconditioner(h, cm.CycleConfig(cm.ChebyshevConfig(cm.Family.fourth, 1, h.lambda_tilde), 4, 0))
        for _ in range(3):
            cm.pgmres(h.A, Mfd, prob.b, None, cm.SolveOptions())
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        f0.record(stream)
        reps = 10
        for _ in range(reps):
            _, frep = cm.pgmres(h.A, Mfd, prob.b, None, cm.SolveOptions())
        f1.record(stream)
        torch.cuda.synchronize()
        fd = {"workload": "FD 5-point n=256 Lx=1 factor 2, PGMRES(30) + 4th-kind (4,0) half V-cycle, tol 1e-6",
              "iterations": frep.iterations, "fine_matvecs": frep.fine_matvecs,
              "time_to_solution_ms": f0.elapsed_time(f1) / reps}
        del h, prob, Mfd
        # FD smoother at HBM scale (n=8192, 48 B/DOF per step + 8 B/DOF for the
        # invD vector the reference passes): bit-exact fused stencil+Chebyshev kernels
        dom = cm.Domain(1.0, 1.0, 8192)
        Af = cm.StencilOperator(dom, ctx)
        invf = cm.jacobi_inverse_diagonal(Af.diagonal(), ctx)
        lt = cm.estimate_lambda_max(Af, invf, 30, 7)
        bf = torch.ones(Af.vec_len(), dtype=torch.float64, device=x.device)
        xf = torch.zeros_like(bf)
        fcfg = cm.ChebyshevConfig(cm.Family.fourth, order, lt)
        for _ in range(3):
            cm.chebyshev_smooth(Af, invf, fcfg, order, bf, xf, False)
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            cm.chebyshev_smooth(Af, invf, fcfg, order, bf, xf, False)
        g1.record(stream)
        torch.cuda.synchronize()
        fms = g0.elapsed_time(g1) / args.steps
        ndof = dom.unknowns()
        # per sweep: residual init (read b, x, invD; write r, d) 40 B, order-2 middle steps
        # (read x, r, d, invD; write x, r, d') 56 B, fused last step (read x, r, d, invD; write x) 40 B
        fd_bytes = (40 + 56 * (order - 2) + 40) * ndof
        fd_gbs = fd_bytes / (fms * 1e-3) / 1e9
        fd["sweep_n8192"] = {
            "workload": "FD 5-point n=8192 (67.1M unknowns) 4th-kind Chebyshev-Jacobi sweep order 8, warm start",
            "value": ndof * order / (fms * 1e-3) / 1e9, "unit": "GDOF-step/s", "ms_per_sweep": fms,
            "roofline": {"bound": "hbm", "achieved": fd_gbs, "peak": peak, "unit": "GB/s", "frac": fd_gbs / peak,
                         "bytes_per_sweep": fd_bytes,
                         "note": "peak is the measured copy (1 read : 1 write) bandwidth; this stream is 4 reads "
                                 ": 3 writes and can exceed it"}}
        del Af, invf, bf, xf
        if not args.no_configs:
            configs = baseline_config_solves(cm, sem, ctx, stream)
        if not args.no_cpu:
            fd["reference_cpu"] = fd_reference_run_case()
            v, kind, sample = cpu_reference_sweeps(args.cpu_E or E, order, 1)
            cpu = {"value": v, "unit": "GDOF-step/s", "cores": 1, "kind": kind, "sample": sample,
                   "cpu": cpu_model(), "host_cores": os.cpu_count()}

    if rank == 0:
        line = {
            "metric": "GDOF/s per Chebyshev smoother sweep", "value": value, "unit": "GDOF-step/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": config_of(E, order, n_glob, world), "partition": f"element z-slabs x{world}",
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "e2e_pipelined": e2e_pipe, "gpu_launches": launches,
            "clocks": clk.summary(), "time_to_solution": tts, "fd_config1": fd, "baseline_configs": configs,
            "setup_s": t_setup, "step_ms_min_max": [min(step_ms), max(step_ms)],
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
