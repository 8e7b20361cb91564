#!/usr/bin/env python3
"""Generate the full-size SEM golden fixtures tests/golden/sem_<case>.json from the
REFERENCE-TEMPLATE CPU path (oracle/_ref, ref_driver.cpp RefPmg):

  the reference's pgmres (krylov.hpp:144-264) preconditioned by its v_cycle
  (multigrid.hpp:69-90) generalised to the p-levels (7,3,1): chebyshev_smooth
  (smoothers.hpp:156-172), residual_into, estimate_lambda_max (:61-79),
  jacobi_inverse_diagonal (:174-181), BandedCholesky (cholesky.hpp:18-91) of
  the assembled p=1 operator; the SEM operator/diagonal/transfers (and the
  Schwarz smoother) from the C restatement oracle/oracle_sem.c, which the GPU
  kernels reproduce bit for bit.

Run HERE (needs /root/reference to build oracle/_ref; single-threaded, the
reference's own contract):

  python oracle/make_golden_sem.py --case E64_box_4th_8_0     # ~1 h, ~42 GB RAM
  python oracle/make_golden_sem.py --case kershaw03_E32       # (8,0) and (4,4)
  python oracle/make_golden_sem.py --case schwarz_E32         # RAS/ASM (2,0), (1,1)

The GPU tests (tests/test_sem_fullsize_gpu.py) rebuild the same right-hand
side with the restatement (orc_sem_rhs; its sha256 is stored) and compare
iteration counts, fine matvecs, residual histories and solution samples.
Floats are hex strings (bit-exact).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_bind as ob  # noqa: E402

# name -> (E, geometry, eps, smoother, [(family, kpre, kpost), ...])
CASES = {
    # BASELINE north_star target: 4th-kind half V-cycle (2k,0), k=4, N=7, E=64^3
    "E64_box_4th_8_0": (64, 0, 1.0, 0, [(2, 8, 0)]),
    # BASELINE configs[3]: deformed (Kershaw eps=0.3) E=32^3, order-2k half vs order-k full
    "kershaw03_E32": (32, 1, 0.3, 0, [(2, 8, 0), (2, 4, 4)]),
    # BASELINE configs[2]: E=32^3 Chebyshev-RAS / -ASM (FDM local solves), 4th kind
    "ras_E32": (32, 0, 1.0, 2, [(2, 2, 0), (2, 1, 1)]),
    "asm_E32": (32, 0, 1.0, 1, [(2, 2, 0), (2, 1, 1)]),
    # small smoke set for checking this script
    "tiny": (3, 1, 0.3, 0, [(2, 4, 0)]),
}
FAMN = {0: "first", 1: "first_opt_lambda", 2: "fourth", 3: "fourth_opt"}
SMN = {0: "jacobi", 1: "asm", 2: "ras"}
N_SAMPLES = 4096


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def sample_idx(n: int) -> np.ndarray:
    return np.unique(np.linspace(0, n - 1, N_SAMPLES).astype(np.int64))


def run(name: str, tol=1e-8, restart=30, maxit=500):
    E, geo, eps, sm, solves = CASES[name]
    t0 = time.time()
    R = ob.RefPmg((7, 3, 1), E, E, E, geo, eps, smoother=sm)
    t_setup = time.time() - t0
    b = R.sem(0).rhs()
    idx = sample_idx(b.size)
    out = {
        "case": name, "orders": [7, 3, 1], "E": [E, E, E], "geometry": geo, "eps": eps, "smoother": SMN[sm],
        "driver": "pgmres", "tol": tol, "restart": restart, "maxit": maxit, "eigen_iterations": 30, "eigen_seed": 7,
        "lambda_max_multiplier": 1.03, "lambda_min_multiplier": 0.1,
        "unknowns": int(b.size), "lambda_tilde": ob.hexs(R.lambda_tilde),
        "rhs": "orc_sem_rhs (PAPER.md:713-715)", "b_sha256": hashlib.sha256(b.tobytes()).hexdigest(),
        "b_norm": float(np.linalg.norm(b)).hex(), "coarse_bandwidth": int(R.R.ref_pmg_coarse_bandwidth(R.h)),
        "x_sample_rule": "unique(linspace(0, n-1, 4096).astype(int64))", "setup_s": t_setup, "cpu": cpu_model(), "cores": 1,
        "generated_by": "oracle/make_golden_sem.py (oracle/_ref RefPmg: reference templates)", "solves": [],
    }
    for fam, kpre, kpost in solves:
        t1 = time.time()
        rep = R.solve(1, fam, kpre, kpost, b, tol=tol, maxit=maxit, restart=restart)
        wall = time.time() - t1
        out["solves"].append({
            "family": FAMN[fam], "k_pre": kpre, "k_post": kpost, "iterations": rep.iterations,
            "fine_matvecs": rep.fine_matvecs, "converged": rep.converged, "status": rep.status,
            "rho": float(rep.rho).hex(), "history": ob.hexs(rep.history),
            "x_norm": float(np.linalg.norm(rep.x)).hex(), "x_samples": ob.hexs(rep.x[idx]), "solve_s": wall,
        })
        print(f"{name} {FAMN[fam]} ({kpre},{kpost}): {rep.iterations} its, {rep.fine_matvecs} mv, "
              f"{rep.status or 'converged'}, {wall:.1f} s", flush=True)
    path = os.path.join(ROOT, "tests", "golden", f"sem_{name}.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=0)
    print("wrote", path, f"({time.time() - t0:.0f} s)", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", action="append", choices=sorted(CASES), required=True)
    a = ap.parse_args()
    for c in a.case:
        run(c)
