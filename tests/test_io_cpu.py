"""Harness text formats (io.hpp) and the sweep/tuning selection logic
(harness.hpp) -- host code, no GPU.  The formatted strings are checked
byte-for-byte against the compiled reference (oracle/_ref) and the cases of
the reference's own test_io.cpp are restated."""
import ctypes as C
import io
import random
import struct

import pytest

import oracle_bind as ob
from paper_2210_03179_b200 import chebmg as cm
from paper_2210_03179_b200 import io as cio


def ref_str(fn, *args):
    buf = C.create_string_buffer(1 << 16)
    n = fn(*args, buf, len(buf))
    assert n < len(buf)
    return buf.value.decode()


@pytest.fixture(scope="module")
def R():
    L = ob.ref()
    L.ref_format_shortest.restype = C.c_size_t
    L.ref_format_shortest.argtypes = [C.c_double, C.c_char_p, C.c_size_t]
    L.ref_beta_table_csv.restype = C.c_size_t
    L.ref_beta_table_csv.argtypes = [C.c_char_p, C.c_size_t]
    L.ref_csv_row.restype = C.c_size_t
    L.ref_csv_row.argtypes = [C.c_double, C.c_size_t, C.c_int, C.c_size_t, C.c_int, C.c_int, C.c_size_t,
                              C.c_size_t, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
                              C.c_double, C.c_int, C.c_char_p, C.c_size_t]
    return L


def _values():
    rng = random.Random(20221007)
    vals = [0.0, -0.0, 1.0, 0.1, 1 / 3, 1.03, 12345.678, 1e-300, 5e-324, 2.0, 1.125, 0.0125, 0.4, 64.0, 128.0,
            1e15, 1e16, 1e17, 1e21, 1e22, 1e23, 123456789012345680000.0, 0.0001, 0.00012, 1e-5, 1.5e-5,
            1.7976931348623157e308, 2.2250738585072014e-308, 21502723.136701405, 0.25, 1.9, 127.25]
    vals += [10.0 ** e for e in range(-30, 31)] + [3.0 * 10.0 ** e for e in range(-25, 26)]
    for _ in range(3000):  # random bit patterns (finite)
        v = struct.unpack("<d", struct.pack("<Q", rng.getrandbits(64)))[0]
        if v == v and abs(v) != float("inf"):
            vals.append(v)
    for _ in range(3000):  # "human" decimals
        vals.append(round(rng.uniform(-1, 1) * 10 ** rng.randint(-8, 12), rng.randint(0, 9)))
    vals += [rng.uniform(0, 2) for _ in range(1000)]
    return vals


def test_format_shortest_matches_reference(R):
    for v in _values():
        mine = cio.format_shortest(v)
        assert mine == ref_str(R.ref_format_shortest, v), v
        assert cio.parse_double(mine) == v or (v != v)
    assert cio.format_shortest(12345) == "12345"  # size_t overload


def test_numeric_parsing_rejects_trailing_junk():  # test_io.cpp:49-56
    assert cio.parse_double("1e3") == 1000.0
    assert cio.parse_size("42") == 42
    for bad in ("1.5x", "", "+1", " 1", "1 ", "0x10", "1_0"):
        with pytest.raises(ValueError):
            cio.parse_double(bad)
    for bad in ("-3", "3.5", "", "+3", "18446744073709551616"):
        with pytest.raises(ValueError):
            cio.parse_size(bad)
    assert cio.parse_size("18446744073709551615") == 2**64 - 1


def test_beta_table_csv_matches_reference(R):
    s = io.StringIO()
    cio.write_beta_table_csv(s)
    out = s.getvalue()
    assert out == ref_str(R.ref_beta_table_csv)
    assert out.startswith("k,i,beta\n") and out.count("\n") == 1 + 210 and "\n1,1,1.125\n" in out


def make_row(family, cycle, **kw):  # test_io.cpp:13-29
    cfg = cm.CaseConfig(Lx=8.0, n=32, factor=2, family=family, k=3, cycle=cycle, driver=cm.Driver.pcg)
    rep = cm.SolveReport(iterations=7, fine_matvecs=56, rho=0.25, converged=True, wall_time_sec=0.0015)
    r = cm.CaseResult(cfg, rep, 1.9)
    for k, v in kw.items():
        setattr(r, k, v)
    return r


def _ref_row(R, r, timing=True):
    return ref_str(R.ref_csv_row, r.cfg.Lx, r.cfg.factor, int(r.cfg.family), r.cfg.k, int(r.cfg.cycle),
                   int(r.cfg.driver), r.report.iterations, r.report.fine_matvecs, r.report.rho,
                   -1.0 if r.C_est is None else r.C_est, r.lambda_tilde, r.cfg.lambda_min_multiplier,
                   -1.0 if r.tuned_lambda_min is None else r.tuned_lambda_min, int(r.report.converged),
                   r.report.wall_time_sec, int(timing))


def test_csv_rows_match_reference(R):
    rng = random.Random(5)
    rows = [make_row(cm.Family.fourth, cm.Cycle.one_sided, C_est=127.25),
            make_row(cm.Family.first, cm.Cycle.full),
            make_row(cm.Family.first_opt_lambda, cm.Cycle.one_sided, tuned_lambda_min=0.0125)]
    for _ in range(200):
        fam = cm.Family(rng.randrange(4))
        r = make_row(fam, cm.Cycle(rng.randrange(2)))
        r.cfg.Lx = rng.choice([1.0, 8.0, 64.0, 128.0, 0.5, 2.75, 1e-3, 1234567.0])
        r.cfg.factor = rng.choice([2, 4, 16])
        r.cfg.k = rng.randint(1, 10)
        r.cfg.driver = cm.Driver(rng.randrange(3))
        r.cfg.lambda_min_multiplier = rng.uniform(0.01, 0.5)
        r.report.iterations = rng.randint(0, 500)
        r.report.fine_matvecs = rng.randint(0, 10000)
        r.report.rho = rng.random()
        r.report.converged = rng.random() < 0.8
        r.report.wall_time_sec = rng.random() * 3
        r.lambda_tilde = rng.uniform(1.9, 2.0)
        r.C_est = rng.uniform(1, 500) if rng.random() < 0.3 else None
        r.tuned_lambda_min = cm.default_tuning_candidates()[rng.randrange(16)] if rng.random() < 0.5 else None
        rows.append(r)
    for r in rows:
        for timing in (True, False):
            assert cio.csv_row(r, cio.CsvOptions(timing)) == _ref_row(R, r, timing)


def test_effective_lambda_min():  # test_io.cpp:58-70
    r = make_row(cm.Family.first, cm.Cycle.full)
    r.cfg.lambda_min_multiplier = 0.15
    assert cio.effective_lambda_min_mult(r) == 0.15
    r = make_row(cm.Family.first_opt_lambda, cm.Cycle.full)
    assert cio.effective_lambda_min_mult(r) is None
    r.tuned_lambda_min = 0.05
    assert cio.effective_lambda_min_mult(r) == 0.05
    assert cio.effective_lambda_min_mult(make_row(cm.Family.fourth, cm.Cycle.full)) is None
    assert cio.effective_lambda_min_mult(make_row(cm.Family.fourth_opt, cm.Cycle.full)) is None


def test_csv_round_trip():  # test_io.cpp:72-111
    rows = [make_row(cm.Family.fourth, cm.Cycle.one_sided, C_est=127.25),
            make_row(cm.Family.first, cm.Cycle.full),
            make_row(cm.Family.first_opt_lambda, cm.Cycle.one_sided, tuned_lambda_min=0.0125)]
    rows[1].report.converged = False
    s = io.StringIO()
    cio.write_csv(s, rows)
    p = cio.parse_csv(io.StringIO(s.getvalue()))
    assert len(p) == 3
    a = p[0]
    assert (a.case_id, a.Lx, a.factor, a.family, a.k_pre, a.k_post, a.cycle, a.driver) == (
        rows[0].cfg.id(), 8.0, 2, "fourth", 6, 0, "one_sided", "pcg")
    assert (a.iterations, a.fine_matvecs, a.rho, a.C_est, a.lambda_tilde) == (7, 56, 0.25, 127.25, 1.9)
    assert a.lambda_min_mult is None and a.converged and a.time_ms == rows[0].report.wall_time_sec * 1e3
    b = p[1]
    assert (b.family, b.k_pre, b.k_post, b.converged, b.C_est) == ("first", 3, 3, False, None)
    assert b.lambda_min_mult == rows[1].cfg.lambda_min_multiplier
    assert p[2].lambda_min_mult == 0.0125


def test_csv_without_timing_and_validation():  # test_io.cpp:113-151
    rows = [make_row(cm.Family.fourth, cm.Cycle.full)]
    a, b = io.StringIO(), io.StringIO()
    cio.write_csv(a, rows)
    cio.write_csv(b, rows, cio.CsvOptions(include_timing=False))
    assert a.getvalue() != b.getvalue() and ",\n" in b.getvalue()
    assert cio.parse_csv(io.StringIO(b.getvalue()))[0].time_ms is None
    for bad in ("", "id,n\n", cio.KCSV_HEADER + "\nonly,three,fields\n",
                cio.KCSV_HEADER + "\nid,1,2,fourth,1,1,full,pcg,1,4,0.5,,1.9,,yes,\n"):
        with pytest.raises(ValueError):
            cio.parse_csv(io.StringIO(bad))
    rows = cio.parse_csv(io.StringIO(cio.KCSV_HEADER + "\r\nid,1,2,fourth,1,1,full,pcg,1,4,0.5,,1.9,,true,\r\n\r\n"))
    assert len(rows) == 1 and rows[0].converged and rows[0].time_ms is None


def test_emit_sweep_csv(tmp_path):
    sr = cm.SweepResult([make_row(cm.Family.fourth, cm.Cycle.full), make_row(cm.Family.fourth, cm.Cycle.one_sided)])
    cm.select_best_rows(sr)
    written = cio.emit_sweep(sr, str(tmp_path))
    assert written == [str(tmp_path) + "/sweep.csv"]
    with open(written[0]) as fh:
        assert len(cio.parse_csv(fh)) == 2
    with pytest.raises(RuntimeError):
        cio.emit_sweep(sr, str(tmp_path / "missing" / "dir"))


def test_config_parse():  # test_io.cpp:200-223
    c = cio.Config.parse(io.StringIO(
        "# leading comment\ncase.n = 64   # trailing comment\ncase.tol = 1e-8\ncase.estimate_c = true\n"
        "sweep.k = 1, 3..5, 9\nsweep.Lx = 1, 8, 64\nsweep.family = fourth , first\n\n"))
    assert c.has("case.n") and not c.has("case.maxit")
    assert c.get_size("case.n", 0) == 64 and c.get_size("case.maxit", 500) == 500
    assert c.get_double("case.tol", 1.0) == 1e-8 and c.get_bool("case.estimate_c", False)
    assert c.get_size_list("sweep.k", []) == [1, 3, 4, 5, 9]
    assert c.get_double_list("sweep.Lx", []) == [1.0, 8.0, 64.0]
    assert c.get_string_list("sweep.family", []) == ["fourth", "first"]
    assert c.unconsumed() == []
    c.reject_unknown()


def test_config_rejects_malformed():  # test_io.cpp:225-244
    for bad in ("case.n 64\n", "a = 1\na = 2\n", " = 3\n"):
        with pytest.raises(cio.ConfigError):
            cio.Config.parse(io.StringIO(bad))
    c = cio.Config.parse(io.StringIO("a = x\nb = 5..2\nc = 1,,2\nd = oui\n"))
    for call in (lambda: c.get_double("a", 0.0), lambda: c.get_size("a", 0), lambda: c.get_size_list("b", []),
                 lambda: c.get_size_list("c", []), lambda: c.get_bool("d", True)):
        with pytest.raises(cio.ConfigError):
            call()
    with pytest.raises(cio.ConfigError):
        cio.Config.parse_file("/nonexistent/chebmg.cfg")
    c = cio.Config.parse(io.StringIO("a = 1\nb = 2\n"))
    assert c.get_size("a", 0) == 1 and c.unconsumed() == ["b"]
    with pytest.raises(cio.ConfigError, match="b"):
        c.reject_unknown()


def test_sweep_spec_from_config():  # test_io.cpp:254-284
    spec = cio.sweep_spec_from_config(cio.Config.parse(io.StringIO(
        "sweep.Lx = 1, 8\nsweep.factor = 2\nsweep.k = 1..3\nsweep.family = fourth_opt\nsweep.cycle = one_sided\n"
        "case.n = 32\ncase.driver = pgmres\ncase.tol = 1e-7\ncase.rhs_seed = 42\n")))
    assert spec.Lx == [1.0, 8.0] and spec.factors == [2] and spec.ks == [1, 2, 3]
    assert spec.families == [cm.Family.fourth_opt] and spec.cycles == [cm.Cycle.one_sided]
    assert (spec.base.n, spec.base.driver, spec.base.tol, spec.base.seeds.rhs, spec.base.maxit) == (
        32, cm.Driver.pgmres, 1e-7, 42, 500)
    for bad in ("sweep.bogus = 1\n", "sweep.family = fifth\n", "case.driver = cg\n"):
        with pytest.raises(cio.ConfigError):
            cio.sweep_spec_from_config(cio.Config.parse(io.StringIO(bad)))


def test_case_id_matches_reference_stream_format():
    c = cm.CaseConfig(Lx=64.0, factor=16, family=cm.Family.fourth_opt, k=9, cycle=cm.Cycle.one_sided,
                      driver=cm.Driver.pgmres)
    assert c.id() == "Lx64_f16_fourth_opt_k9_one_sided_pgmres"
    assert cm.CaseConfig(Lx=0.5).id().startswith("Lx0.5_f2_fourth_k1_one_sided_pcg")
    assert cm.CaseConfig(Lx=1234567.0).id().startswith("Lx1.23457e+06_")


def _rep(its, mv, conv=True):
    return cm.SolveReport(iterations=its, fine_matvecs=mv, converged=conv)


def test_select_tuned():  # harness.hpp:205-217
    rows = [cm.TuneRow(0.1, _rep(5, 50, False)), cm.TuneRow(0.2, _rep(7, 70)), cm.TuneRow(0.3, _rep(6, 66)),
            cm.TuneRow(0.4, _rep(6, 60)), cm.TuneRow(0.5, _rep(6, 60))]
    assert cm.select_tuned(rows) == 3
    assert cm.select_tuned([cm.TuneRow(0.1, _rep(1, 1, False))]) == 1


def test_select_best_rows_and_merge():  # harness.hpp:278-295
    def row(Lx, k, its, mv, conv=True):
        r = make_row(cm.Family.fourth, cm.Cycle.full)
        r.cfg.Lx, r.cfg.k = Lx, k
        r.report = _rep(its, mv, conv)
        return r

    sr = cm.SweepResult([row(1, 3, 5, 30), row(1, 2, 6, 30), row(1, 1, 2, 10, False), row(1, 4, 6, 30),
                         row(8, 1, 9, 90), row(8, 2, 9, 90)])
    cm.select_best_rows(sr)
    assert sr.best_per_group == {(1, 2): 0, (8, 2): 4}
    # rank-split sweep reassembles in reference order
    spec = cm.SweepSpec(Lx=[1.0, 8.0, 64.0], factors=[2], families=[cm.Family.fourth], ks=[1, 2], cycles=[cm.Cycle.full])
    groups = cm.sweep_groups(spec)
    full = [row(Lx, k, k, 10 * k) for (Lx, _f) in groups for k in spec.ks]
    per_rank = [cm.SweepResult([r for gi, (Lx, _f) in enumerate(groups) if gi % 2 == rank
                                for r in full if r.cfg.Lx == Lx]) for rank in range(2)]
    merged = cm.merge_sweep(spec, per_rank)
    assert [(r.cfg.Lx, r.cfg.k) for r in merged.rows] == [(r.cfg.Lx, r.cfg.k) for r in full]
