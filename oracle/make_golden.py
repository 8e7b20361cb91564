#!/usr/bin/env python3
"""Generate tests/golden/*.json from the COMPILED REFERENCE (oracle/_ref).

Run here (where /root/reference exists and oracle/_ref/libchebmg_ref.so is
built by `make -C oracle`):  python oracle/make_golden.py
The fixtures are committed; nothing at test time needs /root/reference.
Floats are stored as hex strings (bit-exact).
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_bind as ob  # noqa: E402

FAM = {"first": 0, "first_opt_lambda": 1, "fourth": 2, "fourth_opt": 3}
DRV = {"pcg": 0, "pgmres": 1, "mg_solver": 2}


def solve_case(n, Lx, f, fam, k_pre, k_post, driver, tol=1e-6):
    """ref_solve on build_problem(rhs_seed=1234) with x0 = 0 -> report + x samples."""
    R = ob.ref()
    h = ob.RefHierarchy(n, Lx, f)
    m = (n - 1) ** 2
    u, b = np.empty(m), np.empty(m)
    R.ref_fd_build_problem(n, Lx, 1.0, 1234, ob.P(u), ob.P(b))
    x0 = np.zeros(m)
    x = np.zeros(m)
    maxit = 500
    hist = np.zeros(maxit + 2)
    hl, its, mv = ob.sz(), ob.sz(), ob.sz()
    cv = C.c_int()
    st = C.create_string_buffer(128)
    rho, wall = C.c_double(), C.c_double()
    t = time.time()
    rc = R.ref_solve(h.h, DRV[driver], FAM[fam], 1.03, 0.1, k_pre, k_post, ob.P(b), ob.P(x0), tol, maxit, 30,
                     ob.P(x), ob.P(hist), maxit + 2, C.byref(hl), C.byref(its), C.byref(mv), C.byref(cv), st,
                     C.byref(rho), C.byref(wall))
    assert rc == 0, R.ref_last_error()
    step = max(1, m // 64)
    return {
        "n": n, "Lx": Lx, "factor": f, "family": fam, "k_pre": k_pre, "k_post": k_post, "driver": driver,
        "tol": tol, "iterations": its.value, "fine_matvecs": mv.value, "converged": bool(cv.value),
        "status": st.value.decode(), "lambda_tilde": h.lambda_tilde.hex(), "rho": rho.value.hex(),
        "history": ob.hexs(hist[: hl.value]), "x_norm": float(np.linalg.norm(x)).hex(),
        "x_stride": step, "x_samples": ob.hexs(x[::step]), "ref_solve_ms": wall.value * 1e3,
        "setup_plus_solve_s": time.time() - t,
    }


def run_case(n, Lx, f, fam, k, cycle, driver):
    h = ob.RefHierarchy(n, Lx, f)
    r = h.run_case(FAM[fam], k, cycle, DRV[driver])
    return {"n": n, "Lx": Lx, "factor": f, "family": fam, "k": k, "cycle": ["full", "one_sided"][cycle],
            "driver": driver, "iterations": r.iterations, "fine_matvecs": r.fine_matvecs,
            "converged": r.converged, "status": r.status, "lambda_tilde": r.lambda_tilde.hex(),
            "tuned_lambda_min": None if r.tuned_lambda_min is None else r.tuned_lambda_min.hex(),
            "history": ob.hexs(r.history), "ref_solve_ms": r.wall_time_sec * 1e3}


def small_vectors():
    """n=16 bit-exact vectors: problem, stencil, transfers, smoother sweeps, V-cycles."""
    R = ob.ref()
    out = {}
    n, Lx = 16, 8.0
    m = (n - 1) ** 2
    u, b = np.empty(m), np.empty(m)
    R.ref_fd_build_problem(n, Lx, 1.0, 1234, ob.P(u), ob.P(b))
    out["problem"] = {"n": n, "Lx": Lx, "seed": 1234, "u": ob.hexs(u), "b": ob.hexs(b)}
    rv = np.empty(50)
    R.ref_random_vector(50, 7, ob.P(rv))
    out["random_vector_seed7_50"] = ob.hexs(rv)
    y = np.empty(m)
    R.ref_fd_stencil_apply(n, Lx, 1.0, ob.P(u), ob.P(y))
    out["stencil_u"] = ob.hexs(y)
    for f in (2, 4):
        mc = (n // f - 1) ** 2
        xc = np.empty(mc)
        R.ref_random_vector(mc, 3, ob.P(xc))
        yp = np.empty(m)
        R.ref_fd_prolong(n, n // f, ob.P(xc), ob.P(yp))
        yr = np.empty(mc)
        R.ref_fd_restrict(n, n // f, ob.P(u), ob.P(yr))
        out[f"prolong_f{f}"] = ob.hexs(yp)
        out[f"restrict_f{f}"] = ob.hexs(yr)
    h = ob.RefHierarchy(n, Lx, 2)
    out["lambda_tilde_n16_Lx8_f2"] = h.lambda_tilde.hex()
    x0 = np.empty(m)
    R.ref_random_vector(m, 13, ob.P(x0))
    sweeps = []
    for fam in FAM:
        for order in (1, 3, 5):
            for xz in (0, 1):
                xin = np.zeros(m) if xz else x0
                x, apps = h.smooth(FAM[fam], order, b, xin, bool(xz))
                sweeps.append({"family": fam, "order": order, "x_is_zero": xz, "apps": apps, "x": ob.hexs(x)})
    out["sweeps"] = sweeps
    cycles = []
    for fam in ("first", "fourth", "fourth_opt"):
        for kp, kq in ((2, 2), (4, 0), (0, 0)):
            x, apps = h.v_cycle(FAM[fam], kp, kq, b, np.zeros(m), True)
            cycles.append({"family": fam, "k_pre": kp, "k_post": kq, "apps": apps, "x": ob.hexs(x)})
    out["v_cycles"] = cycles
    return out


def main():
    os.makedirs(os.path.join(ROOT, "tests", "golden"), exist_ok=True)
    gold = {"generator": "oracle/make_golden.py via oracle/_ref/libchebmg_ref.so (unmodified reference "
                         "headers /root/reference/proj/include, g++ -O2 -std=c++20)"}
    t0 = time.time()
    gold["small"] = small_vectors()
    # SURVEY.md §8c anchor cases + BASELINE.md §3.2 (PGMRES, config 1) + Table 2 under PCG
    solves = []
    for (n, Lx, f, fam, kp, kq, drv) in [
        (256, 1.0, 2, "fourth", 4, 0, "pgmres"),
        (256, 64.0, 2, "fourth", 4, 0, "pgmres"),
        (256, 64.0, 16, "fourth_opt", 8, 0, "pgmres"),
        (256, 128.0, 2, "fourth_opt", 4, 0, "pgmres"),
        (256, 1.0, 16, "fourth", 4, 0, "pgmres"),
        (256, 8.0, 2, "fourth", 4, 0, "pgmres"),
        (256, 8.0, 16, "fourth", 4, 0, "pgmres"),
        (256, 1.0, 2, "fourth", 2, 2, "pgmres"),
        (256, 1.0, 2, "first", 4, 0, "pgmres"),
        (256, 8.0, 16, "fourth", 8, 0, "pgmres"),
        (128, 64.0, 2, "fourth", 18, 0, "pcg"),
        (128, 128.0, 16, "fourth_opt", 18, 0, "pcg"),
        (128, 8.0, 2, "first", 3, 3, "pcg"),
        (128, 8.0, 2, "fourth", 4, 0, "mg_solver"),
    ]:
        solves.append(solve_case(n, Lx, f, fam, kp, kq, drv))
        print(f"solve {n} {Lx} f{f} {fam} ({kp},{kq}) {drv}: its {solves[-1]['iterations']} "
              f"mv {solves[-1]['fine_matvecs']}  {solves[-1]['setup_plus_solve_s']:.1f}s", flush=True)
    gold["solves"] = solves
    cases = []
    for (n, Lx, f, fam, k, cyc, drv) in [  # acceptance.cpp:91-105 rows, PCG default driver
        (128, 1.0, 2, "first_opt_lambda", 2, 0, "pcg"),
        (128, 8.0, 2, "fourth", 7, 1, "pcg"),
        (128, 64.0, 2, "fourth", 9, 1, "pcg"),
        (128, 128.0, 2, "fourth_opt", 9, 1, "pcg"),
        (128, 1.0, 16, "fourth", 8, 1, "pcg"),
        (128, 128.0, 16, "fourth_opt", 9, 1, "pcg"),
    ]:
        cases.append(run_case(n, Lx, f, fam, k, cyc, drv))
        print(f"case {n} {Lx} f{f} {fam} k{k}: its {cases[-1]['iterations']} mv {cases[-1]['fine_matvecs']}",
              flush=True)
    gold["table2_pcg"] = cases
    h = ob.RefHierarchy(128, 8.0, 2)
    gold["estimate_C_n128_Lx8_f2_m20_seed7"] = ob.ref().ref_estimate_C(h.h, 20, 7).hex()
    with open(os.path.join(ROOT, "tests", "golden", "fd_golden.json"), "w") as fh:
        json.dump(gold, fh, indent=1)
    print(f"done in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
