"""The reference-side binding (integration/chebmg_b200_adapter.hpp), compiled
against the UNMODIFIED reference headers into oracle/_ref/libchebmg_adapter.so:
the reference's own templates (chebyshev_smooth, pcg, pgmres, run_case_with)
run with every operator / preconditioner apply on the GPU, and must reproduce
the reference's CPU results.

  - chebyshev_smooth over B200Operator is BITWISE the reference sweep on the CPU
    operator (FD: the stencil kernel is bit-exact; SEM: the operator is bitwise
    the restatement's), for every family / order / x_is_zero.
  - pgmres / pcg over B200Operator + the GPU V-cycle: iteration and matvec
    counts exact, histories within 1e-10 per entry (FD) / 1e-12 ||r0|| (SEM).
  - run_case_with_b200 (dispatch_driver swapped for the device driver,
    harness.hpp:152-168): the reference run_case's counts, histories and tuned
    lambda_min.
"""
import ctypes as C

import numpy as np
import pytest

import oracle_bind as ob

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (ob.adapter_available() and ob.ref_available()),
                                 reason="oracle/_ref adapter not built (make -C oracle in the build container)")]


def test_adapter_fd_smooth_bitwise():
    n, Lx = 64, 1.0
    R = ob.ref()
    h = ob.RefHierarchy(n, Lx, 2)
    m = (n - 1) ** 2
    b = ob.random_vector(m, 3)
    x0 = ob.random_vector(m, 4)
    for fam in (0, 1, 2, 3):
        for order, xz in ((1, True), (4, True), (5, False), (8, False)):
            xr = np.zeros(m) if xz else x0.copy()
            xg = xr.copy()
            apps_r, apps_g = ob.sz(), ob.sz()
            assert R.ref_smooth(h.h, fam, order, h.lambda_tilde, 1.03, 0.1, ob.P(b), ob.P(xr), int(xz),
                                C.byref(apps_r)) == 0
            assert ob.adapter().ad_fd_smooth(n, Lx, fam, order, h.lambda_tilde, ob.P(b), ob.P(xg), int(xz),
                                             C.byref(apps_g)) == 0, ob.adapter().ad_last_error()
            assert apps_g.value == apps_r.value
            assert np.array_equal(xg, xr), (fam, order, xz)


@pytest.mark.parametrize("n,Lx,f,fam,kpre,kpost,driver", [(256, 1.0, 2, 2, 4, 0, 1), (64, 4.0, 2, 3, 2, 2, 0),
                                                          (128, 1.0, 4, 0, 2, 2, 1), (64, 1.0, 2, 2, 6, 0, 1)])
def test_adapter_fd_templates_solve(n, Lx, f, fam, kpre, kpost, driver):
    """reference pcg/pgmres template + B200Operator + GPU V-cycle vs the all-CPU reference."""
    m = (n - 1) ** 2
    h = ob.RefHierarchy(n, Lx, f)
    u, b = ob.build_problem(n, Lx, 1.0, 1234)
    R = ob.ref()
    xr, hist = np.zeros(m), np.zeros(502)
    hl, its, mv = ob.sz(), ob.sz(), ob.sz()
    cv = C.c_int()
    st = C.create_string_buffer(128)
    rho, wall = C.c_double(), C.c_double()
    assert R.ref_solve(h.h, driver, fam, 1.03, 0.1, kpre, kpost, ob.P(b), ob.P(np.zeros(m)), 1e-6, 500, 30,
                       ob.P(xr), ob.P(hist), 502, C.byref(hl), C.byref(its), C.byref(mv), C.byref(cv), st,
                       C.byref(rho), C.byref(wall)) == 0
    g = ob.adapter_report(ob.adapter().ad_fd_solve_templates, n, Lx, f, fam, kpre, kpost, driver, 1e-6, n=m)
    assert (g.iterations, g.fine_matvecs, g.status) == (its.value, mv.value, st.value.decode())
    hr = hist[: hl.value]
    assert np.max(np.abs(np.array(g.history) - hr) / hr) <= 1e-10
    assert np.linalg.norm(g.x - xr) <= 1e-10 * np.linalg.norm(xr)


@pytest.mark.parametrize("fam,k,cycle,driver", [(2, 2, 1, 1), (3, 1, 0, 0), (1, 1, 1, 1), (0, 2, 0, 2),
                                                (2, 1, 1, 0)])
def test_adapter_run_case_b200(fam, k, cycle, driver):
    """run_case_with_b200 (harness with dispatch_driver_b200) vs the reference run_case_with."""
    n, Lx, f = 128, 1.0, 2
    ref = ob.RefHierarchy(n, Lx, f).run_case(fam, k, cycle, driver)
    tuned = C.c_double()
    g = ob.adapter_report(ob.adapter().ad_fd_run_case_b200, n, Lx, f, fam, k, cycle, driver, 1e-6,
                          extra=(C.byref(tuned),))
    assert (g.iterations, g.fine_matvecs, g.converged, g.status) == (ref.iterations, ref.fine_matvecs,
                                                                      ref.converged, ref.status)
    hr = np.array(ref.history)
    assert np.max(np.abs(np.array(g.history) - hr) / hr) <= 1e-10
    if fam == 1:
        assert tuned.value == ref.tuned_lambda_min


@pytest.fixture(scope="module")
def sem_pair():
    R = ob.RefPmg((7, 3, 1), 4, 4, 4)
    h = ob.adapter().ad_pmg_create(4, 0, 1.0, 0)
    assert h, ob.adapter().ad_last_error()
    yield R, h
    ob.adapter().ad_pmg_destroy(h)


def test_adapter_sem_smooth_bitwise(sem_pair):
    R, h = sem_pair
    n = R.n[0]
    b = ob.random_vector(n, 3)
    x0 = ob.random_vector(n, 4)
    for fam in (0, 1, 2, 3):
        for order, xz in ((1, True), (4, True), (8, False)):
            xr, apps_r = R.smooth(0, fam, order, b, np.zeros(n) if xz else x0, xz)
            xg = np.zeros(n) if xz else x0.copy()
            apps = ob.sz()
            assert ob.adapter().ad_pmg_smooth(h, fam, order, R.lambda_tilde[0], ob.P(b), ob.P(xg), int(xz),
                                              C.byref(apps)) == 0, ob.adapter().ad_last_error()
            assert apps.value == apps_r
            assert np.array_equal(xg, xr), (fam, order, xz)


@pytest.mark.parametrize("fam,kpre,kpost,driver", [(2, 8, 0, 1), (0, 4, 4, 1), (2, 2, 2, 0)])
def test_adapter_sem_templates_solve(sem_pair, fam, kpre, kpost, driver):
    """reference pgmres/pcg template + B200Operator(SEM, slot map) + GPU p-MG cycle vs RefPmg."""
    R, h = sem_pair
    b = R.sem(0).rhs()
    ref = R.solve(driver, fam, kpre, kpost, b, tol=1e-8)
    g = ob.adapter_report(ob.adapter().ad_pmg_solve, h, driver, fam, kpre, kpost, ob.P(b), 1e-8, n=R.n[0])
    assert (g.iterations, g.fine_matvecs, g.status) == (ref.iterations, ref.fine_matvecs, ref.status)
    hr = np.array(ref.history)
    d = np.abs(np.array(g.history) - hr)
    print(f"\n[adapter sem {fam} ({kpre},{kpost})] max|h-h_ref|/h0 = {np.max(d) / hr[0]:.3e}, "
          f"per-entry {np.max(d / hr):.3e}")
    assert np.max(d) <= 1e-12 * hr[0]
    assert np.linalg.norm(g.x - ref.x) <= 1e-10 * np.linalg.norm(ref.x)
