"""Pin the CPU restatement (oracle/liboracle.so) to the reference.

1. Against the committed golden fixtures (generated from the compiled,
   unmodified reference by oracle/make_golden.py): bit-exact.
2. Against the live reference build (oracle/_ref) when it is present: bit-exact
   on extra configurations.
CPU only.
"""
import numpy as np
import pytest

import oracle_bind as ob

FAM = {"first": 0, "first_opt_lambda": 1, "fourth": 2, "fourth_opt": 3}
DRV = {"pcg": 0, "pgmres": 1, "mg_solver": 2}


def test_random_vector_bits(golden):
    assert np.array_equal(ob.random_vector(50, 7), ob.unhex(golden["small"]["random_vector_seed7_50"]))


def test_problem_stencil_bits(golden):
    g = golden["small"]["problem"]
    u, b = ob.build_problem(g["n"], g["Lx"], 1.0, g["seed"])
    assert np.array_equal(u, ob.unhex(g["u"]))
    assert np.array_equal(b, ob.unhex(g["b"]))
    assert np.array_equal(ob.stencil_apply(g["n"], g["Lx"], 1.0, u), ob.unhex(golden["small"]["stencil_u"]))


@pytest.mark.parametrize("f", [2, 4])
def test_transfer_bits(golden, f):
    import ctypes as C

    g = golden["small"]["problem"]
    n = g["n"]
    u = ob.unhex(g["u"])
    mc = (n // f - 1) ** 2
    xc = ob.random_vector(mc, 3)
    yp = np.empty((n - 1) ** 2)
    ob.oracle().orc_fd_prolong(n, n // f, ob.P(xc), ob.P(yp))
    yr = np.empty(mc)
    ob.oracle().orc_fd_restrict(n, n // f, ob.P(u), ob.P(yr))
    assert np.array_equal(yp, ob.unhex(golden["small"][f"prolong_f{f}"]))
    assert np.array_equal(yr, ob.unhex(golden["small"][f"restrict_f{f}"]))


def test_smoother_sweeps_bits(golden):
    s = golden["small"]
    b = ob.unhex(s["problem"]["b"])
    h = ob.OracleHierarchy(16, 8.0, 2)
    assert h.lambda_tilde.hex() == s["lambda_tilde_n16_Lx8_f2"]
    x0 = ob.random_vector(h.nf, 13)
    for sw in s["sweeps"]:
        xin = np.zeros(h.nf) if sw["x_is_zero"] else x0
        x = h.smooth(FAM[sw["family"]], sw["order"], b, xin, bool(sw["x_is_zero"]))
        assert np.array_equal(x, ob.unhex(sw["x"])), sw["family"]


def test_v_cycles_bits(golden):
    s = golden["small"]
    b = ob.unhex(s["problem"]["b"])
    h = ob.OracleHierarchy(16, 8.0, 2)
    for cy in s["v_cycles"]:
        x = h.v_cycle(FAM[cy["family"]], cy["k_pre"], cy["k_post"], b, np.zeros(h.nf), True)
        assert np.array_equal(x, ob.unhex(cy["x"]))


def test_table2_rows_exact(golden):
    """acceptance.cpp:91-105 rows under the reference's PCG default: identical bits."""
    for c in golden["table2_pcg"]:
        h = ob.OracleHierarchy(c["n"], c["Lx"], c["factor"])
        r = h.run_case(FAM[c["family"]], c["k"], 0 if c["cycle"] == "full" else 1, DRV[c["driver"]])
        assert (r.iterations, r.fine_matvecs) == (c["iterations"], c["fine_matvecs"])
        assert r.lambda_tilde.hex() == c["lambda_tilde"]
        assert ob.hexs(r.history) == c["history"]
        if c["tuned_lambda_min"] is not None:
            assert r.tuned_lambda_min.hex() == c["tuned_lambda_min"]


def test_solves_exact(golden):
    """SURVEY §8c anchor cases + BASELINE config 1: identical its/mv/histories."""
    for c in golden["solves"]:
        h = ob.OracleHierarchy(c["n"], c["Lx"], c["factor"])
        assert h.lambda_tilde.hex() == c["lambda_tilde"]
        k = c["k_pre"] if c["k_post"] == 0 else c["k_pre"]
        cycle = 1 if c["k_post"] == 0 else 0
        kk = c["k_pre"] // 2 if cycle == 1 else c["k_pre"]
        r = h.run_case(FAM[c["family"]], kk, cycle, DRV[c["driver"]], tol=c["tol"])
        assert (r.iterations, r.fine_matvecs, r.converged) == (c["iterations"], c["fine_matvecs"], c["converged"])
        assert ob.hexs(r.history) == c["history"]
        if r.x is not None and c["driver"] != "mg_solver":
            assert ob.hexs(r.x[:: c["x_stride"]]) == c["x_samples"]
        del k


@pytest.mark.skipif(not ob.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("cfg", [
    (64, 8.0, 2, "fourth", 2, 1, "pgmres"),
    (64, 32.0, 4, "fourth_opt", 3, 0, "pcg"),
    (96, 2.0, 8, "first", 2, 0, "pgmres"),
    (64, 16.0, 2, "first_opt_lambda", 1, 0, "pcg"),
    (64, 4.0, 2, "fourth", 3, 1, "mg_solver"),
])
def test_live_reference_bits(cfg):
    n, Lx, f, fam, k, cyc, drv = cfg
    a = ob.OracleHierarchy(n, Lx, f).run_case(FAM[fam], k, cyc, DRV[drv])
    b = ob.RefHierarchy(n, Lx, f).run_case(FAM[fam], k, cyc, DRV[drv])
    assert (a.iterations, a.fine_matvecs, a.status) == (b.iterations, b.fine_matvecs, b.status)
    assert ob.hexs(a.history) == ob.hexs(b.history)
    assert a.lambda_tilde == b.lambda_tilde


@pytest.mark.skipif(not ob.ref_available(), reason="oracle/_ref not built")
def test_live_reference_coarse_solve_bits():
    a = ob.OracleHierarchy(64, 8.0, 2)
    b = ob.RefHierarchy(64, 8.0, 2)
    assert ob.oracle().orc_fd_hier_bandwidth(a.h) == ob.ref().ref_hier_bandwidth(b.h)
    rc = ob.random_vector(a.nc, 5)
    ea = a.coarse_solve(rc)
    eb = np.empty_like(rc)
    ob.ref().ref_hier_coarse_solve(b.h, ob.P(rc), ob.P(eb))
    assert np.array_equal(ea, eb)


def test_beta_table_known_values():
    """test_beta.cpp:27-33 spot values and the order-1 closed form."""
    L = ob.oracle()
    assert L.orc_beta_coefficients(1)[0] == 1.125
    assert not L.orc_beta_coefficients(21)
    assert not L.orc_beta_coefficients(0)
    for k in range(1, 21):
        row = [L.orc_beta_coefficients(k)[i] for i in range(k)]
        assert all(row[i] < row[i + 1] for i in range(k - 1))  # strictly increasing (beta_table.hpp:13)
