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
