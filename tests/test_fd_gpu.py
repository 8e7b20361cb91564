"""FD path parity on the GPU: CUDA library (through the C-ABI) vs the oracle /
the reference's golden fixtures.

Bit-exact: stencil, transfers, Chebyshev sweeps (all families), operator
counts.  Within 1e-10 relative: V-cycles (separable FDM coarse solve instead
of banded Cholesky) and Krylov histories / solutions (tree-ordered inner
products).  Iteration counts and fine_matvecs: exact.
"""
import numpy as np
import pytest
import torch

import oracle_bind as ob

pytestmark = pytest.mark.gpu

FAM = {"first": 0, "first_opt_lambda": 1, "fourth": 2, "fourth_opt": 3}
TOL_REL = 1e-10  # BASELINE.json north_star: "within 1e-10 relative in fp64"


@pytest.fixture(scope="module")
def cm():
    from paper_2210_03179_b200 import chebmg

    return chebmg


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


def host(t):
    return t.detach().cpu().numpy()


def test_stencil_bits(cm, golden):
    g = golden["small"]["problem"]
    A = cm.StencilOperator(cm.Domain(g["Lx"], 1.0, g["n"]))
    u = dev(ob.unhex(g["u"]))
    y = A.new_vector()
    A.apply(u, y)
    assert np.array_equal(host(y), ob.unhex(golden["small"]["stencil_u"]))
    assert A.applications() == 1
    assert np.all(host(A.diagonal()) == 2.0 * (1.0 / (8.0 / 16) ** 2 + 1.0 / (1.0 / 16) ** 2))
    # large grid vs oracle restatement
    n, Lx = 1024, 3.0
    x = ob.random_vector((n - 1) ** 2, 9)
    A2 = cm.StencilOperator(cm.Domain(Lx, 1.0, n))
    y2 = A2.new_vector()
    A2.apply(dev(x), y2)
    assert np.array_equal(host(y2), ob.stencil_apply(n, Lx, 1.0, x))


@pytest.mark.parametrize("f", [2, 4])
def test_transfer_bits(cm, golden, f):
    g = golden["small"]["problem"]
    n = g["n"]
    h = cm.build_hierarchy(cm.Domain(g["Lx"], 1.0, n), f)
    xc = ob.random_vector((n // f - 1) ** 2, 3)
    assert np.array_equal(host(h.prolong(dev(xc))), ob.unhex(golden["small"][f"prolong_f{f}"]))
    assert np.array_equal(host(h.restrict(dev(ob.unhex(g["u"])))), ob.unhex(golden["small"][f"restrict_f{f}"]))


def test_lambda_tilde_and_sweeps_bits(cm, golden):
    """Every Chebyshev sweep is bit-identical to the reference (smoothers.hpp:95-172),
    and costs k-1 matvecs from zero, k warm (test_smoothers.cpp:69-88)."""
    s = golden["small"]
    h = cm.build_hierarchy(cm.Domain(8.0, 1.0, 16), 2)
    # power iteration: tree-ordered dots, so near (not bit) equal
    lt_ref = float.fromhex(s["lambda_tilde_n16_Lx8_f2"])
    assert abs(h.lambda_tilde - lt_ref) <= 1e-13 * lt_ref
    b = dev(ob.unhex(s["problem"]["b"]))
    x0 = ob.random_vector(h.fine_dim(), 13)
    invd = h.inv_diag
    for sw in s["sweeps"]:
        cfg = cm.ChebyshevConfig(cm.Family(FAM[sw["family"]]), sw["order"], lt_ref)
        x = torch.zeros_like(b) if sw["x_is_zero"] else dev(x0)
        h.A.reset_applications()
        cm.chebyshev_smooth(h.A, invd, cfg, sw["order"], b, x, bool(sw["x_is_zero"]))
        assert h.A.applications() == sw["apps"]
        assert np.array_equal(host(x), ob.unhex(sw["x"])), (sw["family"], sw["order"], sw["x_is_zero"])


def test_smoother_errors(cm):
    h = cm.build_hierarchy(cm.Domain(1.0, 1.0, 8), 2)
    b = h.A.new_vector()
    x = h.A.new_vector()
    with pytest.raises(IndexError):
        cm.chebyshev_smooth(h.A, h.inv_diag, cm.ChebyshevConfig(cm.Family.fourth_opt, 21, 1.9), 21, b, x, True)
    with pytest.raises(ValueError):
        cm.chebyshev_smooth(h.A, h.inv_diag, cm.ChebyshevConfig(cm.Family.first, 2, 1.9, 1.0, 1.5), 2, b, x, True)
    # order 0 is a no-op that skips validation (smoothers.hpp:159)
    cm.chebyshev_smooth(h.A, h.inv_diag, cm.ChebyshevConfig(cm.Family.first, 0, -1.0), 0, b, x, True)
    with pytest.raises(ValueError):
        cm.build_hierarchy(cm.Domain(8.0, 1.0, 16), 3)


@pytest.mark.parametrize("n,Lx,f", [(16, 8.0, 2), (64, 1.0, 2), (256, 64.0, 16), (256, 128.0, 2)])
def test_coarse_solve_matches_cholesky(cm, n, Lx, f):
    """Separable FDM coarse solve == the reference's banded Cholesky (cholesky.hpp:44-58)."""
    h = cm.build_hierarchy(cm.Domain(Lx, 1.0, n), f)
    oh = ob.OracleHierarchy(n, Lx, f)
    rc = ob.random_vector(oh.nc, 21)
    e_ref = oh.coarse_solve(rc)
    e = host(h.coarse_solve(dev(rc)))
    assert np.max(np.abs(e - e_ref)) <= 1e-12 * np.max(np.abs(e_ref))


def test_v_cycles(cm, golden):
    s = golden["small"]
    h = cm.build_hierarchy(cm.Domain(8.0, 1.0, 16), 2)
    lt_ref = float.fromhex(s["lambda_tilde_n16_Lx8_f2"])
    b = dev(ob.unhex(s["problem"]["b"]))
    for cy in s["v_cycles"]:
        cfg = cm.CycleConfig(cm.ChebyshevConfig(cm.Family(FAM[cy["family"]]), 1, lt_ref), cy["k_pre"], cy["k_post"])
        h.A.reset_applications()
        z = cm.preconditioner_apply(h, cfg, b)
        assert h.A.applications() == cy["apps"] == cy["k_pre"] + cy["k_post"]
        ref = ob.unhex(cy["x"])
        assert np.max(np.abs(host(z) - ref)) <= TOL_REL * np.max(np.abs(ref))


def test_preconditioner_cost_2k(cm):
    """test_multigrid.cpp:115-130: every application costs exactly 2k fine matvecs."""
    h = cm.build_hierarchy(cm.Domain(64.0, 1.0, 32), 2)
    v = dev(ob.random_vector(h.fine_dim(), 31))
    for fam in (cm.Family.first, cm.Family.fourth, cm.Family.fourth_opt):
        s = cm.ChebyshevConfig(fam, 1, h.lambda_tilde, 1.0, 0.1)
        for k in range(1, 11):
            h.A.reset_applications()
            cm.preconditioner_apply(h, cm.full_cycle(s, k), v)
            assert h.A.applications() == 2 * k
            h.A.reset_applications()
            cm.preconditioner_apply(h, cm.one_sided_cycle(s, k), v)
            assert h.A.applications() == 2 * k


def _check_solve(c, rep, x=None):
    assert rep.iterations == c["iterations"], (c, rep.iterations)
    assert rep.fine_matvecs == c["fine_matvecs"]
    assert rep.converged == c["converged"]
    assert rep.status == c["status"]
    href = ob.unhex(c["history"])
    h = np.array(rep.residual_history)
    assert h.shape == href.shape
    assert np.max(np.abs(h - href) / href) <= TOL_REL
    if x is not None:
        xs = host(x)[:: c["x_stride"]]
        xr = ob.unhex(c["x_samples"])
        assert np.max(np.abs(xs - xr)) <= TOL_REL * float.fromhex(c["x_norm"])


def test_golden_solves(cm, golden):
    """SURVEY §8c anchors and BASELINE config 1 (n=256 PGMRES half V-cycle)."""
    for c in golden["solves"]:
        h = cm.build_hierarchy(cm.Domain(c["Lx"], 1.0, c["n"]), c["factor"])
        lt = float.fromhex(c["lambda_tilde"])
        assert abs(h.lambda_tilde - lt) <= 1e-12 * lt
        prob = cm.build_problem(h.domain, 1234)
        cfg = cm.CycleConfig(cm.ChebyshevConfig(cm.Family(FAM[c["family"]]), 1, h.lambda_tilde), c["k_pre"],
                             c["k_post"])
        M = cm.vcycle_preconditioner(h, cfg)
        opts = cm.SolveOptions(tol=c["tol"])
        if c["driver"] == "pgmres":
            x, rep = cm.pgmres(h.A, M, prob.b, None, opts)
        elif c["driver"] == "pcg":
            x, rep = cm.pcg(h.A, M, prob.b, None, opts)
        else:
            x, rep = None, cm.stationary_solve(h.A, M, prob.b, c["tol"], 500)
        _check_solve(c, rep, x)


def test_table2_run_case(cm, golden):
    """acceptance.cpp:91-105 rows through the Python harness mirror (run_case)."""
    for c in golden["table2_pcg"]:
        cfg = cm.CaseConfig(Lx=c["Lx"], n=c["n"], factor=c["factor"], family=cm.Family(FAM[c["family"]]), k=c["k"],
                            cycle=cm.Cycle.full if c["cycle"] == "full" else cm.Cycle.one_sided,
                            driver=cm.Driver.pcg)
        r = cm.run_case(cfg)
        assert (r.report.iterations, r.report.fine_matvecs) == (c["iterations"], c["fine_matvecs"])
        href = ob.unhex(c["history"])
        assert np.max(np.abs(np.array(r.report.residual_history) - href) / href) <= TOL_REL
        if c["tuned_lambda_min"] is not None:
            assert r.tuned_lambda_min == float.fromhex(c["tuned_lambda_min"])


def test_live_oracle_more_configs(cm):
    """Seeded configurations beyond the fixtures vs the restatement (== reference bits)."""
    for (n, Lx, f, fam, k, cyc, drv) in [(128, 32.0, 4, "fourth_opt", 3, 1, "pgmres"),
                                        (64, 2.0, 8, "first", 2, 0, "pgmres"),
                                        (128, 16.0, 2, "fourth", 5, 1, "pcg"),
                                        (96, 4.0, 2, "fourth", 2, 0, "mg_solver")]:
        oref = ob.OracleHierarchy(n, Lx, f).run_case(FAM[fam], k, cyc, {"pcg": 0, "pgmres": 1, "mg_solver": 2}[drv])
        cfg = cm.CaseConfig(Lx=Lx, n=n, factor=f, family=cm.Family(FAM[fam]), k=k, cycle=cm.Cycle(cyc),
                            driver=cm.Driver[drv])
        r = cm.run_case(cfg)
        assert (r.report.iterations, r.report.fine_matvecs, r.report.status) == (
            oref.iterations, oref.fine_matvecs, oref.status)
        h = np.array(r.report.residual_history)
        assert np.max(np.abs(h - np.array(oref.history)) / np.array(oref.history)) <= TOL_REL


def test_identity_pcg_and_zero_rhs(cm):
    """test_krylov.cpp: plain CG to 1e-10; zero RHS converges immediately."""
    A = cm.StencilOperator(cm.Domain(1.0, 1.0, 8))
    b = dev(ob.random_vector(A.rows(), 3))
    M = cm.identity_preconditioner()
    x, rep = cm.pcg(A, M, b, None, cm.SolveOptions(tol=1e-10, maxit=400))
    assert rep.converged and rep.status == ""
    assert len(rep.residual_history) == rep.iterations + 1
    assert rep.rho < 1.0
    Ad = np.stack([ob.stencil_apply(8, 1.0, 1.0, e) for e in np.eye(A.rows())], axis=1)
    xr = np.linalg.solve(Ad, host(b))
    assert np.linalg.norm(host(x) - xr) < 1e-8 * np.linalg.norm(xr)
    z = torch.zeros_like(b)
    for fn in (cm.pcg, cm.pgmres):
        x, rep = fn(A, M, z, None, cm.SolveOptions())
        assert rep.converged and rep.status == "zero initial residual" and rep.iterations == 0


def test_python_callable_preconditioner_and_symmetry_probe(cm):
    h = cm.build_hierarchy(cm.Domain(1.0, 1.0, 16), 2)
    s = cm.ChebyshevConfig(cm.Family.first, 1, h.lambda_tilde)
    prob = cm.build_problem(h.domain, 9)
    # full cycle passes the symmetry probe (test_krylov.cpp: "full-cycle ... passes")
    M = cm.vcycle_preconditioner(h, cm.CycleConfig(s, 2, 2))
    x, rep = cm.pcg(h.A, M, prob.b, None, cm.SolveOptions(enforce_spd_preconditioner=True))
    assert rep.converged

    def skew(v):
        y = v.clone()
        y[0] += 0.5 * v[1]
        return y

    with pytest.raises(ValueError):
        cm.pcg(h.A, skew, prob.b, None, cm.SolveOptions(enforce_spd_preconditioner=True))


def test_determinism(cm):
    cfg = cm.CaseConfig(Lx=64.0, n=128, factor=2, family=cm.Family.fourth, k=2, driver=cm.Driver.pgmres)
    a = cm.run_case(cfg).report.residual_history
    b = cm.run_case(cfg).report.residual_history
    assert a == b


def test_estimate_C_golden(cm, golden):
    """lanczos.hpp:97-155 on the device vs the reference's C (golden, n=128 Lx=8 f=2 m=20 seed=7).
    The exact fine solve is a fast-diagonalisation solve instead of the banded
    Cholesky, so C agrees to rounding of the Lanczos recurrence, not bitwise."""
    h = cm.build_hierarchy(cm.Domain(8.0, 1.0, 128), 2)
    est = cm.estimate_C(h, 20, 7)
    ref = float.fromhex(golden["estimate_C_n128_Lx8_f2_m20_seed7"])
    assert est.m == 20 and len(est.alpha) == 20 and len(est.beta) == 19
    assert abs(est.C - ref) <= 1e-9 * ref, (est.C, ref)


@pytest.mark.parametrize("n,Lx,f,m,seed", [(32, 1.0, 2, 8, 3), (64, 16.0, 4, 20, 99), (128, 1.0, 8, 12, 5)])
def test_estimate_C_live_reference(cm, n, Lx, f, m, seed):
    h = cm.build_hierarchy(cm.Domain(Lx, 1.0, n), f)
    rh = ob.RefHierarchy(n, Lx, f)
    ref = ob.ref().ref_estimate_C(rh.h, m, seed)
    est = cm.estimate_C(h, m, seed)
    assert abs(est.C - ref) <= 1e-9 * ref, (est.C, ref)
    with pytest.raises(ValueError):
        cm.estimate_C(h, 0)


def test_concurrent_tuning_identical_to_sequential(cm):
    """harness.hpp:186-201: the 16 lambda_min candidate solves run concurrently
    (one stream + hierarchy clone each) and give the sequential reports exactly."""
    cfg = cm.CaseConfig(Lx=1.0, n=64, factor=2, family=cm.Family.first_opt_lambda, k=2, cycle=cm.Cycle.full)
    h = cm.build_hierarchy(cm.Domain(1.0, 1.0, 64), 2)
    cands = cm.default_tuning_candidates()
    seq = cm.tune_lambda_min_table(cfg, h, cands, concurrent=False)
    par = cm.tune_lambda_min_table(cfg, h, cands, concurrent=True)
    for a, b in zip(seq, par):
        assert a.candidate == b.candidate
        assert (a.report.iterations, a.report.fine_matvecs, a.report.converged) == (
            b.report.iterations, b.report.fine_matvecs, b.report.converged)
        assert a.report.residual_history == b.report.residual_history
    assert cm.select_tuned(seq) == cm.select_tuned(par)


def _ref_sweep_rows(cfg_text):
    import ctypes as C
    import io as _io

    from paper_2210_03179_b200 import io as cio

    L = ob.ref()
    L.ref_sweep_csv.restype = C.c_int
    L.ref_sweep_csv.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
    buf = C.create_string_buffer(1 << 20)
    n = C.c_size_t()
    assert L.ref_sweep_csv(cfg_text.encode(), buf, len(buf), C.byref(n)) == 0, ob.ref().ref_last_error()
    return cio.parse_csv(_io.StringIO(buf.value.decode()))


def test_sweep_csv_matches_reference_sweep(cm, tmp_path):
    """The reference's sweep (harness.hpp:297-337) and ours on the same config
    text: identical rows (ids, counts, convergence, lambda_tilde bits, tuned
    lambda_min, C) with rho / C within the fp64 tolerance; the best row per
    group is the same."""
    import io as _io

    from paper_2210_03179_b200 import io as cio

    text = ("sweep.Lx = 1, 64\nsweep.factor = 2, 4\nsweep.k = 1..3\n"
            "sweep.family = first, first_opt_lambda, fourth, fourth_opt\nsweep.cycle = full, one_sided\n"
            "case.n = 32\ncase.driver = pgmres\ncase.tol = 1e-8\ncase.estimate_c = true\n")
    ref = _ref_sweep_rows(text)
    spec = cio.sweep_spec_from_config(cio.Config.parse(_io.StringIO(text)))
    sr = cm.sweep(spec)
    out = cio.emit_sweep(sr, str(tmp_path), opts=cio.CsvOptions(include_timing=False))
    with open(out[0]) as fh:
        mine = cio.parse_csv(fh)
    assert len(mine) == len(ref) == 2 * 2 * 4 * 3 * 2
    for a, b in zip(mine, ref):
        assert (a.case_id, a.Lx, a.factor, a.family, a.k_pre, a.k_post, a.cycle, a.driver) == (
            b.case_id, b.Lx, b.factor, b.family, b.k_pre, b.k_post, b.cycle, b.driver)
        assert (a.iterations, a.fine_matvecs, a.converged, a.lambda_min_mult) == (
            b.iterations, b.fine_matvecs, b.converged, b.lambda_min_mult), a.case_id
        # power-iteration norms are tree-reduced on the device: lambda_tilde to rounding
        assert abs(a.lambda_tilde - b.lambda_tilde) <= 1e-13 * b.lambda_tilde
        # rho = (h_N/h_0)^(1/N): the histories agree to 1e-10 h_0, i.e. h_N only to
        # ~1e-10 h_0/h_N ~ 1e-2 relative at tol 1e-8, divided by N in rho
        assert abs(a.rho - b.rho) <= 1e-6 * b.rho
        assert abs(a.C_est - b.C_est) <= 1e-9 * b.C_est
        assert a.time_ms is None
    # best row per (Lx, factor): fewest matvecs, then iterations, then k
    ref_sr = cm.SweepResult([cm.CaseResult(r.cfg, cm.SolveReport(b.iterations, b.fine_matvecs, converged=b.converged))
                             for r, b in zip(sr.rows, ref)])
    cm.select_best_rows(ref_sr)
    assert ref_sr.best_per_group == sr.best_per_group


@pytest.mark.parametrize("restart", [30, 63, 64, 70, 100, 200])
def test_pgmres_any_restart_matches_reference(cm, restart):
    """krylov.hpp:148 accepts any restart >= 1: above 63 the Arnoldi scalars move to a
    restart-sized workspace, the least-squares solve to dynamic shared (or global)
    memory and the multi-dots / updates / iterate run in 64-vector chunks with the
    same per-entry order.  84 PGMRES iterations (n=128, Lx=64, 1st kind k=1),
    so restarts 30..70 restart and 100/200 do not -- vs the compiled reference."""
    n, Lx, f = 128, 64.0, 2
    ref = ob.RefHierarchy(n, Lx, f).run_case(0, 1, 1, 1, restart=restart)
    cfg = cm.CaseConfig(Lx=Lx, n=n, factor=f, family=cm.Family.first, k=1, cycle=cm.Cycle.one_sided,
                        driver=cm.Driver.pgmres, restart=restart)
    r = cm.run_case(cfg)
    assert (r.report.iterations, r.report.fine_matvecs, r.report.status) == (ref.iterations, ref.fine_matvecs,
                                                                             ref.status)
    h, hr = np.array(r.report.residual_history), np.array(ref.history)
    assert np.max(np.abs(h - hr) / hr) <= TOL_REL


def test_pgmres_restart_zero_rejected(cm):
    cfg = cm.CaseConfig(n=32, driver=cm.Driver.pgmres, restart=0)
    with pytest.raises(ValueError, match="restart must be >= 1"):
        cm.run_case(cfg)
