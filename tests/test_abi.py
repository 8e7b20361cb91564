"""The C-ABI library loads and exports every symbol include/chebmg_b200.h declares;
host-only entry points agree with the reference bit-for-bit.  CPU only (no
compute call touches a GPU here)."""
import ctypes as C

import numpy as np

import oracle_bind as ob


def test_library_exports_every_header_symbol():
    from paper_2210_03179_b200 import _lib

    declared = _lib.header_symbols()
    assert len(declared) > 40
    missing = [s for s in declared if not hasattr(_lib.lib, s)]
    assert missing == [], missing
    assert _lib.missing == [], _lib.missing


def test_version_and_errors():
    from paper_2210_03179_b200 import _lib

    assert b"sm_100a" in _lib.lib.cmg_version()
    out = (C.c_double * 4)()
    assert _lib.lib.cmg_beta_coefficients(21, out) == _lib.CMG_ERANGE
    assert b"outside tabulated range" in _lib.lib.cmg_last_error()


def test_host_random_vector_bits(golden):
    from paper_2210_03179_b200 import chebmg as cm

    assert np.array_equal(cm.random_vector(50, 7), ob.unhex(golden["small"]["random_vector_seed7_50"]))


def test_host_build_problem_bits(golden):
    from paper_2210_03179_b200 import chebmg as cm

    g = golden["small"]["problem"]
    u, b = cm.build_problem_host(cm.Domain(g["Lx"], 1.0, g["n"]), g["seed"])
    assert np.array_equal(u, ob.unhex(g["u"]))
    assert np.array_equal(b, ob.unhex(g["b"]))
    # config-1 size: identical to the oracle restatement
    u2, b2 = cm.build_problem_host(cm.Domain(1.0, 1.0, 256), 1234)
    uo, bo = ob.build_problem(256, 1.0, 1.0, 1234)
    assert np.array_equal(u2, uo) and np.array_equal(b2, bo)


def test_beta_coefficients_match_oracle():
    from paper_2210_03179_b200 import chebmg as cm

    for k in range(1, 21):
        row = cm.beta_coefficients(k)
        orow = ob.oracle().orc_beta_coefficients(k)
        assert row == [orow[i] for i in range(k)]
    try:
        cm.beta_coefficients(0)
        raise AssertionError("expected IndexError")
    except IndexError:
        pass


def test_domain_validation():
    from paper_2210_03179_b200 import chebmg as cm

    for bad in [dict(Lx=1.0, Ly=1.0, n=1), dict(Lx=0.0, Ly=1.0, n=8)]:
        try:
            cm.Domain(**bad)
            raise AssertionError("expected ValueError")
        except ValueError:
            pass


def _dp(a):
    return a.ctypes.data_as(C.c_void_p)


def test_sem_host_tables_bitwise_equal_oracle():
    """The GLL basis, derivative and interpolation matrices and the 1D Schwarz
    FDM bases the device operators are built from are bit-identical to the
    restatement's (oracle_sem.c / oracle_schwarz.c) -- the precondition for the
    bitwise operator/transfer/local-solve comparisons in the -m gpu tests."""
    from paper_2210_03179_b200 import _lib

    L = ob.oracle()
    ob._sem_protos(L)
    L.orc_fdm_1d.argtypes = [C.c_int, ob.dp, ob.dp, ob.dp, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
                             C.c_int, C.c_int, ob.dp, ob.dp]
    for N in range(1, 8):
        xi, w, D = np.empty(N + 1), np.empty(N + 1), np.empty((N + 1) ** 2)
        assert _lib.lib.cmg_sem_basis_host(N, _dp(xi), _dp(w), _dp(D)) == 0
        oxi, ow, oD = ob.gll(N)
        assert xi.tobytes() == oxi.tobytes() and w.tobytes() == ow.tobytes()
        assert D.tobytes() == oD.reshape(-1).tobytes()
        for Nc in range(1, N + 1):
            J = np.empty((N + 1) * (Nc + 1))
            assert _lib.lib.cmg_sem_interp_host(N, Nc, _dp(J)) == 0
            assert J.tobytes() == ob.interp_matrix(N, Nc).reshape(-1).tobytes()
    for N in (2, 3, 5, 7):
        xi, w, D = ob.gll(N)
        D = np.ascontiguousarray(D.reshape(-1))
        for lens in ((0.1, 0.1, 0.1), (0.07, 0.13, 0.21)):
            for flags in ((0, 0, 0, 0), (1, 1, 0, 0), (1, 0, 0, 0), (0, 0, 1, 1), (0, 0, 0, 1)):
                S, lam = np.empty((N + 3) ** 2), np.empty(N + 3)
                oS, olam = np.empty((N + 3) ** 2), np.empty(N + 3)
                assert _lib.lib.cmg_sem_fdm1d_host(N, *lens, *flags, _dp(S), _dp(lam)) == 0
                L.orc_fdm_1d(N, ob.P(xi), ob.P(w), ob.P(D), *lens, *flags, ob.P(oS), ob.P(olam))
                assert S.tobytes() == oS.tobytes() and lam.tobytes() == olam.tobytes(), (N, lens, flags)
