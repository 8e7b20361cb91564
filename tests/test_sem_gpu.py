"""SEM p-multigrid path on the GPU vs the restatement (oracle/oracle_sem.c) and the
reference's own templates driving it (oracle/_ref RefPmg: pgmres, chebyshev_smooth,
residual_into, estimate_lambda_max, BandedCholesky).

Bitwise: the operator, its diagonal, the p-transfers, Chebyshev sweeps at a given
lambda and the Schwarz local solves -- the GPU kernels and the restatement share
one arithmetic contract (k_sem.cu / oracle_sem.c headers: explicit fma chains,
no other contraction).

Solves: iteration counts and fine_matvecs exact; solutions within 1e-10
relative (BASELINE north_star); residual histories entrywise within
1e-12 * ||r_0|| -- or, on a GMRES plateau, within 10x of the floor two equally
exact CPU paths show against each other (the restated C drivers vs the
reference templates, which differ only in the coarse-matrix assembly order).
The per-entry relative error is printed: it cannot reach 1e-10 at the tail of
a 1e-8-converged history, because the reference's own sequential dot products
carry ~1e-14 relative rounding, which enters the iterate and hence the true
residual at 1e-14 * ||b||, i.e. 1e-6 relative to a 1e-8 * ||b|| residual
(DESIGN.md §5)."""
import numpy as np
import pytest
import torch

import oracle_bind as ob

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def cm():
    from paper_2210_03179_b200 import chebmg

    return chebmg


@pytest.fixture(scope="module")
def sem():
    from paper_2210_03179_b200 import sem

    return sem


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


def same(a, b):
    """bitwise equality (up to the sign of zero)"""
    return np.array_equal(np.asarray(a), np.asarray(b))


def check_history(h, hr, floor=0.0, what=""):
    h, hr = np.asarray(h), np.asarray(hr)
    assert h.size == hr.size
    d = np.abs(h - hr)
    per_entry = float(np.max(d / hr))
    print(f"\n[{what}] history: max|h-h_ref|/h0 = {np.max(d) / hr[0]:.3e}, max per-entry rel = {per_entry:.3e}, "
          f"CPU-vs-CPU floor/h0 = {floor / hr[0]:.3e}")
    assert np.max(d) <= max(1e-12 * hr[0], 10.0 * floor)
    return per_entry


def check_x(x, xr, what="", floor=0.0):
    """x within 1e-10 relative, or within 10x a measured CPU-vs-CPU floor (relative)"""
    e = float(np.linalg.norm(x - xr) / np.linalg.norm(xr))
    print(f"[{what}] x rel err = {e:.3e} (CPU-vs-CPU floor {floor:.3e})")
    assert e <= max(TOL, 10.0 * floor)


@pytest.mark.parametrize("N,ex,ey,ez,geo", [(7, 3, 2, 4, 0), (7, 2, 3, 2, 1), (3, 4, 3, 2, 0), (1, 5, 4, 3, 0),
                                            (5, 2, 2, 3, 1), (2, 3, 3, 3, 0), (4, 3, 2, 3, 1), (3, 2, 3, 4, 1)])
def test_apply_diag_rhs(sem, N, ex, ey, ez, geo):
    d = sem.SemDesc(N, ex, ey, ez, geometry=geo, eps=0.3)
    A = sem.SemOperator(d)
    o = ob.OracleSem(N, ex, ey, ez, geo, 0.3)
    assert A.rows() == o.n
    x = ob.random_vector(o.n, 17)
    y = A.new_vector()
    A.apply(A.from_canonical(x), y)
    assert A.applications() == 1
    assert same(A.to_canonical(y), o.apply(x))
    assert same(A.to_canonical(A.diagonal()), o.diagonal())
    assert rel(A.to_canonical(A.rhs()), o.rhs()) <= 1e-12  # device sin(): not bitwise
    # padding slots stay exactly zero
    assert torch.all(y.cpu()[torch.from_numpy(~A.valid)] == 0)


def test_sweeps_all_families(cm, sem):
    d = sem.SemDesc(7, 3, 2, 2, geometry=1, eps=0.3)
    P = sem.PMGHierarchy(d, (7, 3, 1))
    o = ob.OraclePmg((7, 3, 1), 3, 2, 2, 1, 0.3)
    for l in (0, 1):
        assert abs(P.lambda_tilde[l] - o.lambda_tilde[l]) <= 1e-11 * o.lambda_tilde[l]
    for lev in (0, 1):  # p=7 (line kernels) and p=3 (packed low-order kernel)
        A = P.ops[lev]
        b = ob.random_vector(o.n[lev], 3)
        x0 = ob.random_vector(o.n[lev], 4)
        for fam in (0, 1, 2, 3):
            for order, xz in ((1, True), (4, True), (5, False), (8, False)):
                cfg = cm.ChebyshevConfig(cm.Family(fam), order, o.lambda_tilde[lev])
                x = A.from_canonical(np.zeros(o.n[lev]) if xz else x0)
                A.reset_applications()
                cm.chebyshev_smooth(A, P.inv_diag(lev), cfg, order, A.from_canonical(b), x, xz)
                assert A.applications() == (order - 1 if xz else order)
                ref = o.smooth(lev, fam, order, b, np.zeros(o.n[lev]) if xz else x0, xz)
                assert same(A.to_canonical(x), ref), (lev, fam, order, xz)


def test_transfers_and_coarse_solve(sem):
    for geo in (0, 1):
        d = sem.SemDesc(7, 4, 3, 3, geometry=geo, eps=0.3)
        P = sem.PMGHierarchy(d, (7, 3, 1))
        o = ob.OraclePmg((7, 3, 1), 4, 3, 3, geo, 0.3)
        for l in (0, 1):
            xc = ob.random_vector(o.n[l + 1], 5)
            xf = ob.random_vector(o.n[l], 6)
            Pc, Pf = P.ops[l + 1], P.ops[l]
            assert same(Pf.to_canonical(P.prolong(l, Pc.from_canonical(xc))), o.prolong(l, xc))
            assert same(Pc.to_canonical(P.restrict(l, Pf.from_canonical(xf))), o.restrict(l, xf))
        rc = ob.random_vector(o.n[2], 7)
        C1 = P.ops[2]
        assert rel(C1.to_canonical(P.coarse_solve(C1.from_canonical(rc))), o.coarse_solve(rc)) <= 1e-11


@pytest.mark.parametrize("fam,kpre,kpost", [(2, 4, 0), (3, 4, 0), (0, 2, 2), (2, 2, 2)])
def test_v_cycle(cm, sem, fam, kpre, kpost):
    d = sem.SemDesc(7, 3, 3, 2)
    P = sem.PMGHierarchy(d, (7, 3, 1))
    o = ob.OraclePmg((7, 3, 1), 3, 3, 2)
    b = o.sem(0).rhs()
    cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family(fam), 1, 1.0), kpre, kpost)
    P.A.reset_applications()
    z = P.preconditioner_apply(cyc, P.A.from_canonical(b))
    assert P.A.applications() == kpre + kpost
    assert rel(P.A.to_canonical(z), o.v_cycle(fam, kpre, kpost, b)) <= TOL


def ref_solve_with_floor(ex, ey, ez, geo, eps, smoother, fam, kpre, kpost, driver=1, floor=True):
    """The reference-template CPU solve (RefPmg) and, optionally, the floor: the
    largest history difference between it and the restated C drivers
    (OraclePmg.solve), an equally exact CPU path."""
    R = ob.RefPmg((7, 3, 1), ex, ey, ez, geo, eps, smoother=smoother)
    b = R.sem(0).rhs()
    ref = R.solve(driver, fam, kpre, kpost, b, tol=1e-8)
    fl = 0.0
    if floor:
        o = ob.OraclePmg((7, 3, 1), ex, ey, ez, geo, eps, smoother=smoother)
        alt = o.solve(driver, fam, kpre, kpost, b, tol=1e-8)
        assert (alt.iterations, alt.fine_matvecs) == (ref.iterations, ref.fine_matvecs)
        fl = float(np.max(np.abs(np.array(alt.history) - np.array(ref.history))))
    return R, b, ref, fl


def gpu_solve(cm, P, fam, kpre, kpost, b, driver=1):
    cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family(fam), 1, P.lambda_tilde[0]), kpre, kpost)
    fn = cm.pgmres if driver == 1 else cm.pcg
    return fn(P.A, P.preconditioner(cyc), P.A.from_canonical(b), None, cm.SolveOptions(tol=1e-8))


@pytest.mark.parametrize("fam,kpre,kpost,driver", [(2, 4, 0, "pgmres"), (3, 4, 0, "pgmres"), (0, 2, 2, "pgmres"),
                                                   (2, 2, 2, "pcg"), (2, 8, 0, "pgmres")])
def test_pmg_solves_match_reference_templates(cm, sem, fam, kpre, kpost, driver):
    """p-MG(7,3,1)-preconditioned PGMRES/PCG (tol 1e-8): GPU vs the
    reference's own pcg/pgmres + v_cycle + chebyshev_smooth templates (RefPmg)."""
    ex, ey, ez = 4, 3, 3
    drv = {"pcg": 0, "pgmres": 1}[driver]
    R, b, ref, fl = ref_solve_with_floor(ex, ey, ez, 0, 1.0, 0, fam, kpre, kpost, drv)
    P = sem.PMGHierarchy(sem.SemDesc(7, ex, ey, ez), (7, 3, 1))
    assert abs(P.lambda_tilde[0] - R.lambda_tilde[0]) <= 1e-12 * R.lambda_tilde[0]
    x, rep = gpu_solve(cm, P, fam, kpre, kpost, b, drv)
    assert (rep.iterations, rep.fine_matvecs, rep.status) == (ref.iterations, ref.fine_matvecs, ref.status)
    check_history(rep.residual_history, ref.history, fl, f"{driver} {fam} ({kpre},{kpost})")
    check_x(P.A.to_canonical(x), ref.x)


def test_indefinite_level_rejected(sem):
    """A Kershaw eps=0.05 map whose z-kink (z = 1/2) falls inside an element
    layer (ez = 9) gives an indefinite interpolated geometry: setup refuses it
    with EINVAL instead of smoothing with a negative lambda_tilde."""
    with pytest.raises(ValueError, match="not positive definite"):
        sem.PMGHierarchy(sem.SemDesc(7, 36, 36, 9, geometry=sem.KERSHAW, eps=0.05), (7, 3, 1))


@pytest.mark.parametrize("eps,kpre,kpost", [(0.3, 4, 0), (0.3, 8, 0), (0.5, 4, 0), (0.5, 2, 2), (0.3, 2, 2)])
def test_kershaw_solves(cm, sem, eps, kpre, kpost):
    """Deformed-mesh config (BASELINE configs[3] shape): half (2k,0) vs full (k,k)
    cycles vs the reference templates.  (0.3, (2,2)) needs 86 PGMRES(30)
    iterations through two restarts and plateaus between iterations ~50 and ~70:
    there the two CPU paths themselves drift apart by ~1e-9 of ||r_0|| (coarse
    assembly order only), so the bound is the measured floor, not 1e-12."""
    ex = ey = ez = 3
    R, b, ref, fl = ref_solve_with_floor(ex, ey, ez, 1, eps, 0, 2, kpre, kpost)
    P = sem.PMGHierarchy(sem.SemDesc(7, ex, ey, ez, geometry=sem.KERSHAW, eps=eps), (7, 3, 1))
    x, rep = gpu_solve(cm, P, 2, kpre, kpost, b)
    assert (rep.iterations, rep.fine_matvecs) == (ref.iterations, ref.fine_matvecs)
    check_history(rep.residual_history, ref.history, fl, f"kershaw {eps} ({kpre},{kpost})")
    check_x(P.A.to_canonical(x), ref.x)


@pytest.mark.parametrize("ras", [0, 1])
@pytest.mark.parametrize("N,geo", [(7, 0), (3, 0), (7, 1)])
def test_schwarz_apply(sem, ras, N, geo):
    """Chebyshev-Schwarz smoother S_ASM / S_RAS vs the oracle."""
    d = sem.SemDesc(N, 3, 2, 3, geometry=geo, eps=0.3)
    orders = (N, 1) if N == 3 else (N, 3, 1)
    P = sem.PMGHierarchy(d, orders, smoother=sem.RAS if ras else sem.ASM)
    o = ob.OracleSem(N, 3, 2, 3, geo, 0.3)
    r = ob.random_vector(o.n, 9)
    out = P.A.new_vector()
    from paper_2210_03179_b200 import _lib
    import ctypes as C

    _lib.check(_lib.lib.cmg_pmg_schwarz_apply(P.h, 0, C.c_void_p(P.A.from_canonical(r).data_ptr()),
                                              C.c_void_p(out.data_ptr())))
    import os

    if os.environ.get("CMG_SCHWARZ_MMA") == "1":  # opt-in DMMA local solve: not bitwise, rounding only
        assert rel(P.A.to_canonical(out), o.schwarz(r, ras)) <= 1e-12
    else:
        assert same(P.A.to_canonical(out), o.schwarz(r, ras))


@pytest.mark.parametrize("smoother,fam,kpre,kpost", [(2, 2, 2, 0), (1, 2, 2, 0), (2, 0, 1, 1), (1, 3, 2, 0),
                                                     (2, 0, 2, 2), (1, 0, 2, 2), (2, 1, 2, 2)])
def test_schwarz_pmg_solves(cm, sem, smoother, fam, kpre, kpost):
    """BASELINE configs[2] shape: Chebyshev-ASM/RAS p-MG(7,3,1) PGMRES (non-symmetric
    smoother); the 1st-kind (2,2) cases run the fused x += d update of the
    Schwarz step (EPI_SUPD1 / asm_emit kind 1) at order 2."""
    ex, ey, ez = 3, 3, 2
    R, b, ref, fl = ref_solve_with_floor(ex, ey, ez, 0, 1.0, smoother, fam, kpre, kpost)
    P = sem.PMGHierarchy(sem.SemDesc(7, ex, ey, ez), (7, 3, 1), smoother=smoother)
    for l in (0, 1):
        assert abs(P.lambda_tilde[l] - R.lambda_tilde[l]) <= 1e-12 * R.lambda_tilde[l]
    x, rep = gpu_solve(cm, P, fam, kpre, kpost, b)
    assert (rep.iterations, rep.fine_matvecs) == (ref.iterations, ref.fine_matvecs)
    check_history(rep.residual_history, ref.history, fl, f"schwarz {smoother} fam {fam} ({kpre},{kpost})")
    check_x(P.A.to_canonical(x), ref.x)


def test_determinism(cm, sem):
    d = sem.SemDesc(7, 3, 3, 3)
    P = sem.PMGHierarchy(d, (7, 3, 1))
    b = P.A.rhs()
    cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family.fourth, 1, P.lambda_tilde[0]), 4, 0)
    r1 = cm.pgmres(P.A, P.preconditioner(cyc), b, None, cm.SolveOptions(tol=1e-8))[1]
    r2 = cm.pgmres(P.A, P.preconditioner(cyc), b, None, cm.SolveOptions(tol=1e-8))[1]
    assert r1.residual_history == r2.residual_history


@pytest.mark.parametrize("smoother,geo", [(0, 0), (2, 0), (1, 0), (0, 1)])
def test_graph_replayed_preconditioner_same_bits_and_counts(cm, sem, smoother, geo):
    """On one GPU the p-MG preconditioner captures each (v, z) pair into a CUDA
    graph after its first apply and replays it (sem.cpp PmgPrecond): the replayed
    solves must give the bits, histories and operator counts of the direct first
    solve (the first apply of each solve and of the object runs directly)."""
    d = sem.SemDesc(7, 4, 3, 3, geometry=geo, eps=0.3)
    P = sem.PMGHierarchy(d, (7, 3, 1), smoother=smoother)
    b = P.A.rhs()
    cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family.fourth, 1, P.lambda_tilde[0]), 2, 1)
    M = P.preconditioner(cyc)
    runs = []
    for _ in range(3):
        P.A.reset_applications()
        x, rep = cm.pgmres(P.A, M, b, None, cm.SolveOptions(tol=1e-10, restart=5, maxit=200))
        runs.append((x.cpu().numpy().tobytes(), rep.residual_history, rep.iterations, rep.fine_matvecs,
                     P.A.applications()))
    assert runs[0][2] > 5  # restarts: the same (v, z) pairs are replayed within a solve too
    assert runs[1] == runs[0] and runs[2] == runs[0]


def test_graph_recaptured_after_workspace_growth(cm, sem):
    """The RAS smoother's scratch is a context workspace slot; a larger hierarchy on
    the same context reallocates it, so the captured V-cycle graphs of the smaller
    one must be recaptured (PmgPrecond::ws_now), not replayed on freed memory."""
    def solver(E):
        P = sem.PMGHierarchy(sem.SemDesc(7, *E), (7, 3, 1), smoother=2)
        M = P.preconditioner(cm.CycleConfig(cm.ChebyshevConfig(cm.Family.fourth, 1, P.lambda_tilde[0]), 1, 1))
        b = P.A.rhs()

        def run():
            x, rep = cm.pgmres(P.A, M, b, None, cm.SolveOptions(tol=1e-10, restart=4, maxit=100))
            return x.cpu().numpy().tobytes(), rep.residual_history
        return P, M, run

    P1, M1, run1 = solver((3, 3, 2))
    first = run1()
    assert run1() == first
    P2, M2, run2 = solver((5, 4, 4))
    run2()
    assert run1() == first
    assert run1() == first


def test_graft_smoke():
    import os
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import __graft_entry__

    __graft_entry__.smoke()


@pytest.fixture(scope="module")
def config1_pair(sem):
    """BASELINE configs[1] at full size: N=7, E=16^3 (1.37M unknowns), p-MG(7,3,1)."""
    if not ob.ref_available():
        pytest.skip("oracle/_ref not built")
    R = ob.RefPmg((7, 3, 1), 16, 16, 16)
    P = sem.PMGHierarchy(sem.SemDesc(7, 16, 16, 16), (7, 3, 1))
    return R, P


@pytest.mark.parametrize("fam,kpre,kpost", [(2, 8, 0), (2, 4, 4), (3, 8, 0), (0, 4, 4), (0, 8, 0), (3, 4, 4)])
def test_config1_full_size_vs_reference(cm, config1_pair, fam, kpre, kpost):
    """configs[1] (E=16^3) half (2k,0) vs full (k,k) cycles, 1st/4th/opt-4th kind:
    PGMRES(30) to 1e-8, GPU vs the reference templates (RefPmg) -- same iteration
    counts, histories within 1e-12 ||r_0||, solutions within 1e-10."""
    R, P = config1_pair
    assert abs(P.lambda_tilde[0] - R.lambda_tilde[0]) <= 1e-12 * R.lambda_tilde[0]
    b = R.sem(0).rhs()
    ref = R.solve(1, fam, kpre, kpost, b, tol=1e-8)
    x, rep = gpu_solve(cm, P, fam, kpre, kpost, b)
    assert (rep.iterations, rep.fine_matvecs, rep.converged) == (ref.iterations, ref.fine_matvecs, True)
    check_history(rep.residual_history, ref.history, 0.0, f"config1 {fam} ({kpre},{kpost})")
    check_x(P.A.to_canonical(x), ref.x)


@pytest.mark.parametrize("restart", [70, 120])
def test_sem_pgmres_restart_above_63(cm, sem, restart):
    """restart > 63 on the SEM path (layer multi-dots in 64-vector chunks): the
    111-iteration Kershaw eps=0.3 (2,0) solve with one restart (70) and none
    (120).  A weak smoother on a deformed mesh stalls on GMRES plateaus, where
    the two exact CPU paths already differ by ~1e-6 ||r0|| in the history and
    ~3e-10 in x, so both bounds are 10x that measured floor."""
    ex = ey = ez = 3
    R = ob.RefPmg((7, 3, 1), ex, ey, ez, 1, 0.3)
    b = R.sem(0).rhs()
    ref = R.solve(1, 2, 2, 0, b, tol=1e-8, restart=restart)
    alt = ob.OraclePmg((7, 3, 1), ex, ey, ez, 1, 0.3).solve(1, 2, 2, 0, b, tol=1e-8, restart=restart)
    floor = float(np.max(np.abs(np.array(alt.history) - np.array(ref.history))))
    floor_x = float(np.linalg.norm(alt.x - ref.x) / np.linalg.norm(ref.x))
    P = sem.PMGHierarchy(sem.SemDesc(7, ex, ey, ez, geometry=sem.KERSHAW, eps=0.3), (7, 3, 1))
    cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family.fourth, 1, P.lambda_tilde[0]), 2, 0)
    x, rep = cm.pgmres(P.A, P.preconditioner(cyc), P.A.from_canonical(b), None,
                       cm.SolveOptions(tol=1e-8, restart=restart))
    assert rep.iterations > 64
    assert (rep.iterations, rep.fine_matvecs, rep.status) == (ref.iterations, ref.fine_matvecs, ref.status)
    check_history(rep.residual_history, ref.history, floor, f"restart {restart}")
    check_x(P.A.to_canonical(x), ref.x, f"restart {restart}", floor_x)


def test_coarse_cg_fallback_under_pgmres_and_pcg_rejected(cm, sem, monkeypatch):
    """Deformed mesh above CMG_COARSE_DENSE_MAX (forced to 0 here): the p=1 solve is
    the tolerance-stopped CG (relative residual 1e-13), a variable preconditioner.
    PGMRES still reproduces the reference template's iteration count and
    solution; PCG refuses it (EINVAL) instead of running without its theory."""
    monkeypatch.setenv("CMG_COARSE_DENSE_MAX", "0")
    ex = ey = ez = 3
    R, b, ref, _ = ref_solve_with_floor(ex, ey, ez, 1, 0.3, 0, 2, 4, 0, floor=False)
    P = sem.PMGHierarchy(sem.SemDesc(7, ex, ey, ez, geometry=sem.KERSHAW, eps=0.3), (7, 3, 1))
    x, rep = gpu_solve(cm, P, 2, 4, 0, b)
    assert (rep.iterations, rep.fine_matvecs) == (ref.iterations, ref.fine_matvecs)
    h, hr = np.array(rep.residual_history), np.array(ref.history)
    print(f"\n[coarse CG] max|h-h_ref|/h0 = {np.max(np.abs(h - hr)) / hr[0]:.3e}")
    assert np.max(np.abs(h - hr)) <= 1e-10 * hr[0]
    check_x(P.A.to_canonical(x), ref.x)
    with pytest.raises(ValueError, match="not a fixed linear operator"):
        gpu_solve(cm, P, 2, 2, 2, b, driver=0)


@pytest.mark.parametrize("geo", [0, 1])
def test_tall_mesh_apply_and_sweeps_bitwise(cm, sem, geo):
    """A taller mesh (12 element layers, 3x2 per layer): operator and sweeps
    bitwise against the restatement on box and Kershaw geometry."""
    ex, ey, ez = 3, 2, 12
    P = sem.PMGHierarchy(sem.SemDesc(7, ex, ey, ez, geometry=geo, eps=0.3), (7, 3, 1))
    o = ob.OraclePmg((7, 3, 1), ex, ey, ez, geo, 0.3)
    A = P.ops[0]
    x = ob.random_vector(o.n[0], 17)
    y = A.new_vector()
    A.apply(A.from_canonical(x), y)
    assert same(A.to_canonical(y), o.sem(0).apply(x))
    b = ob.random_vector(o.n[0], 3)
    for fam in (0, 2, 3):
        for order, xz in ((4, True), (8, False)):
            cfg = cm.ChebyshevConfig(cm.Family(fam), order, o.lambda_tilde[0])
            xd = A.from_canonical(np.zeros(o.n[0]) if xz else x)
            cm.chebyshev_smooth(A, P.inv_diag(0), cfg, order, A.from_canonical(b), xd, xz)
            ref = o.smooth(0, fam, order, b, np.zeros(o.n[0]) if xz else x, xz)
            assert same(A.to_canonical(xd), ref), (fam, order, xz)


@pytest.mark.parametrize("E", [(1, 1, 1), (2, 1, 1), (1, 2, 3)])
def test_degenerate_meshes_empty_coarse_level(cm, sem, E):
    """One-element-thick meshes: the p=1 level has no interior unknowns (an empty
    coarse solve), the p=3 level a handful -- counts and histories as the
    reference templates (which accept an empty BandedCholesky)."""
    R, b, ref, _ = ref_solve_with_floor(*E, 0, 1.0, 0, 2, 4, 0, floor=False)
    assert R.n[2] == 0
    P = sem.PMGHierarchy(sem.SemDesc(7, *E), (7, 3, 1))
    x, rep = gpu_solve(cm, P, 2, 4, 0, b)
    assert (rep.iterations, rep.fine_matvecs, rep.status) == (ref.iterations, ref.fine_matvecs, ref.status)
    check_history(rep.residual_history, ref.history, 0.0, f"mesh {E}")
    check_x(P.A.to_canonical(x), ref.x, f"mesh {E}")


@pytest.mark.parametrize("case", ["zero_rhs", "maxit", "restart1", "pcg"])
def test_sem_solver_edge_cases(cm, sem, case):
    """krylov.hpp edge paths on the SEM operator vs the reference templates: a zero
    right-hand side ("zero initial residual", x = 0), maxit reached mid-cycle,
    restart = 1 (every iteration restarts), PCG with a symmetric (2,2) cycle."""
    ex = ey = ez = 3
    R = ob.RefPmg((7, 3, 1), ex, ey, ez)
    b = np.zeros(R.n[0]) if case == "zero_rhs" else R.sem(0).rhs()
    drv, kpre, kpost, kw = 1, 4, 0, {}
    if case == "maxit":
        kw = {"maxit": 3}
    elif case == "restart1":
        kw = {"restart": 1}
    elif case == "pcg":
        drv, kpre, kpost = 0, 2, 2
    ref = R.solve(drv, 2, kpre, kpost, b, tol=1e-8, **kw)
    P = sem.PMGHierarchy(sem.SemDesc(7, ex, ey, ez), (7, 3, 1))
    cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family.fourth, 1, P.lambda_tilde[0]), kpre, kpost)
    fn = cm.pgmres if drv == 1 else cm.pcg
    x, rep = fn(P.A, P.preconditioner(cyc), P.A.from_canonical(b), None, cm.SolveOptions(tol=1e-8, **kw))
    assert (rep.iterations, rep.fine_matvecs, rep.status, rep.converged) == (
        ref.iterations, ref.fine_matvecs, ref.status, ref.converged)
    if case == "zero_rhs":
        assert rep.residual_history == [0.0] and not np.any(P.A.to_canonical(x))
        return
    check_history(rep.residual_history, ref.history, 0.0, case)
    check_x(P.A.to_canonical(x), ref.x, case)
