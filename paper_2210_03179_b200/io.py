"""Result and configuration formats of the reference harness (io.hpp).

Host-side text formats only -- the same 16-column sweep CSV, the beta-table
dump and the flat ``key = value`` config files -- so rows produced by the GPU
runs diff byte-for-byte against the reference CLI's output:

* ``format_shortest``      io.hpp:27-37   (std::to_chars shortest round trip)
* ``parse_double/size``    io.hpp:39-53   (std::from_chars, whole string)
* ``KCSV_HEADER``          io.hpp:55-57
* ``write_csv_row/csv``    io.hpp:65-90
* ``CsvRow``/``parse_csv`` io.hpp:92-172
* ``write_beta_table_csv`` io.hpp:174-182
* ``emit_sweep`` (csv)     io.hpp:335-365
* ``Config``               io.hpp:382-523
* ``sweep_spec_from_config`` io.hpp:525-563

The SVG plots of io.hpp:184-333 are presentation, outside the hot-path scope
(SURVEY.md §8f row 4 names the CSV and config formats).
"""
from __future__ import annotations

import math
import re
from dataclasses import dataclass
from typing import IO, Iterable, List, Optional

from .chebmg import (BETA_MAX_ORDER, CaseResult, Family, SweepResult, SweepSpec, beta_coefficients,
                     cycle_from_string, driver_from_string, family_from_string)

# ---------------------------------------------------------------- numbers


def format_shortest(v) -> str:
    """``std::to_chars(double)`` without a format: the shortest digit string that
    parses back to the same double, written in fixed or scientific notation,
    whichever is shorter (fixed on a tie).  Integers print as integers."""
    if isinstance(v, bool):
        raise TypeError("format_shortest: bool")
    if isinstance(v, int):
        return str(v)
    v = float(v)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    if v == 0.0:
        return sign + "0"
    r = repr(abs(v))  # CPython: shortest round-trip digits (correctly rounded)
    mant, _, exp = r.partition("e")
    ip, _, fp = mant.partition(".")
    alld = ip + fp  # value = 0.alld * 10^(len(ip) + exp)
    stripped = alld.lstrip("0")
    P = len(ip) + (int(exp) if exp else 0) - (len(alld) - len(stripped))
    digits = stripped.rstrip("0")
    E = P - 1  # scientific exponent: value = d.ddd * 10^E
    # fixed notation
    if E >= 0:
        # an integral value in fixed notation prints its exact integer digits
        # (printf %f semantics), e.g. 123456789012345683968 for 1.2345678901234568e+20
        fixed = str(int(abs(v))) if len(digits) <= E + 1 else digits[:E + 1] + "." + digits[E + 1:]
    else:
        fixed = "0." + "0" * (-E - 1) + digits
    sci = digits[0] + ("." + digits[1:] if len(digits) > 1 else "") + "e" + ("+" if E >= 0 else "-") + f"{abs(E):02d}"
    return sign + (fixed if len(fixed) <= len(sci) else sci)


_DOUBLE_RE = re.compile(r"-?(?:(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|inf(?:inity)?|nan(?:\([A-Za-z0-9_]*\))?)",
                        re.IGNORECASE)


def parse_double(s: str) -> float:
    """io.hpp:39-45: std::from_chars over the whole string (no sign '+', no spaces)."""
    if not _DOUBLE_RE.fullmatch(s):
        raise ValueError(f"not a number: '{s}'")
    return float(s)


def parse_size(s: str) -> int:
    """io.hpp:47-53: std::from_chars into size_t over the whole string."""
    if not re.fullmatch(r"\d+", s) or int(s) >= 2**64:
        raise ValueError(f"not a nonnegative integer: '{s}'")
    return int(s)


# ---------------------------------------------------------------- CSV

KCSV_HEADER = ("case_id,L_x,factor,family,k_pre,k_post,cycle,driver,iterations,fine_matvecs,"
               "rho,C_est,lambda_tilde,lambda_min_mult,converged,time_ms")


@dataclass
class CsvOptions:  # io.hpp:59-63
    include_timing: bool = True


def effective_lambda_min_mult(r: CaseResult) -> Optional[float]:  # io.hpp:65-69
    if r.cfg.family == Family.first:
        return r.cfg.lambda_min_multiplier
    if r.cfg.family == Family.first_opt_lambda:
        return r.tuned_lambda_min
    return None


def csv_row(r: CaseResult, opts: CsvOptions = CsvOptions()) -> str:
    """One CSV record, newline included (io.hpp:71-84)."""

    def opt(v):
        return "" if v is None else format_shortest(v)

    f = [r.cfg.id(), format_shortest(r.cfg.Lx), str(r.cfg.factor), r.cfg.family.name, str(r.cfg.k_pre()),
         str(r.cfg.k_post()), r.cfg.cycle.name, r.cfg.driver.name, str(r.report.iterations),
         str(r.report.fine_matvecs), format_shortest(r.report.rho), opt(r.C_est), format_shortest(r.lambda_tilde),
         opt(effective_lambda_min_mult(r)), "true" if r.report.converged else "false",
         format_shortest(r.report.wall_time_sec * 1e3) if opts.include_timing else ""]
    return ",".join(f) + "\n"


def write_csv_row(os_: IO[str], r: CaseResult, opts: CsvOptions = CsvOptions()) -> None:
    os_.write(csv_row(r, opts))


def write_csv(os_: IO[str], rows: Iterable[CaseResult], opts: CsvOptions = CsvOptions()) -> None:
    """io.hpp:86-90."""
    os_.write(KCSV_HEADER + "\n")
    for r in rows:
        write_csv_row(os_, r, opts)


@dataclass
class CsvRow:  # io.hpp:93-111
    case_id: str = ""
    Lx: float = 0.0
    factor: int = 0
    family: str = ""
    k_pre: int = 0
    k_post: int = 0
    cycle: str = ""
    driver: str = ""
    iterations: int = 0
    fine_matvecs: int = 0
    rho: float = 0.0
    C_est: Optional[float] = None
    lambda_tilde: float = 0.0
    lambda_min_mult: Optional[float] = None
    converged: bool = False
    time_ms: Optional[float] = None


def _opt_field(s: str) -> Optional[float]:
    return None if s == "" else parse_double(s)


def parse_csv(is_: IO[str]) -> List[CsvRow]:
    """io.hpp:136-172."""
    lines = is_.read().split("\n")
    if lines and lines[-1] == "":
        lines.pop()  # getline does not yield a record after the final newline
    if not lines:
        raise ValueError("parse_csv: empty input")
    head = lines[0][:-1] if lines[0].endswith("\r") else lines[0]
    if head != KCSV_HEADER:
        raise ValueError("parse_csv: unexpected header: " + head)
    rows = []
    for line in lines[1:]:
        if line.endswith("\r"):
            line = line[:-1]
        if not line:
            continue
        f = line.split(",")
        if len(f) != 16:
            raise ValueError(f"parse_csv: expected 16 fields, got {len(f)}")
        if f[14] not in ("true", "false"):
            raise ValueError("parse_csv: bad converged field: " + f[14])
        rows.append(CsvRow(f[0], parse_double(f[1]), parse_size(f[2]), f[3], parse_size(f[4]), parse_size(f[5]),
                           f[6], f[7], parse_size(f[8]), parse_size(f[9]), parse_double(f[10]), _opt_field(f[11]),
                           parse_double(f[12]), _opt_field(f[13]), f[14] == "true", _opt_field(f[15])))
    return rows


def write_beta_table_csv(os_: IO[str]) -> None:
    """io.hpp:174-182: k,i,beta for every tabulated order."""
    os_.write("k,i,beta\n")
    for k in range(1, BETA_MAX_ORDER + 1):
        for i, b in enumerate(beta_coefficients(k), start=1):
            os_.write(f"{k},{i},{format_shortest(b)}\n")


def emit_sweep(sr: SweepResult, out_dir: str, want_csv: bool = True, opts: CsvOptions = CsvOptions()) -> List[str]:
    """io.hpp:335-365, CSV part: writes out_dir/sweep.csv, returns the paths written."""
    written = []
    if want_csv:
        path = out_dir + "/sweep.csv"
        try:
            fh = open(path, "w", newline="")
        except OSError:
            raise RuntimeError("cannot open " + path) from None
        with fh:
            write_csv(fh, sr.rows, opts)
        written.append(path)
    return written


# ---------------------------------------------------------------- config files


class ConfigError(RuntimeError):  # io.hpp:370-373
    pass


def _trim(s: str) -> str:  # io.hpp:377-382 (std::isspace, "C" locale)
    return s.strip(" \t\n\v\f\r")


class Config:
    """Flat dotted-key configuration (io.hpp:388-523): ``key = value`` lines,
    ``#`` starts a comment; accessors record the keys they read."""

    def __init__(self):
        self._kv: dict[str, str] = {}
        self._consumed: set[str] = set()

    @staticmethod
    def parse(is_: IO[str]) -> "Config":
        c = Config()
        text = is_.read()
        lines = text.split("\n")
        if lines and lines[-1] == "":
            lines.pop()
        for lineno, line in enumerate(lines, start=1):
            h = line.find("#")
            if h >= 0:
                line = line[:h]
            line = _trim(line)
            if not line:
                continue
            eq = line.find("=")
            if eq < 0:
                raise ConfigError(f"config line {lineno}: expected key = value")
            key, value = _trim(line[:eq]), _trim(line[eq + 1:])
            if not key:
                raise ConfigError(f"config line {lineno}: empty key")
            if key in c._kv:
                raise ConfigError(f"config line {lineno}: duplicate key {key}")
            c._kv[key] = value
        return c

    @staticmethod
    def parse_file(path: str) -> "Config":
        try:
            fh = open(path)
        except OSError:
            raise ConfigError("cannot open config file " + path) from None
        with fh:
            return Config.parse(fh)

    def has(self, key: str) -> bool:
        return key in self._kv

    def get_string(self, key: str, default: str) -> str:
        self._consumed.add(key)
        return self._kv.get(key, default)

    def get_double(self, key: str, default: float) -> float:
        self._consumed.add(key)
        if key not in self._kv:
            return default
        try:
            return parse_double(self._kv[key])
        except ValueError:
            raise ConfigError(f"config key {key}: not a number: {self._kv[key]}") from None

    def get_size(self, key: str, default: int) -> int:
        self._consumed.add(key)
        if key not in self._kv:
            return default
        try:
            return parse_size(self._kv[key])
        except ValueError:
            raise ConfigError(f"config key {key}: not an integer: {self._kv[key]}") from None

    def get_bool(self, key: str, default: bool) -> bool:
        self._consumed.add(key)
        if key not in self._kv:
            return default
        v = self._kv[key]
        if v == "true":
            return True
        if v == "false":
            return False
        raise ConfigError(f"config key {key}: expected true or false, got {v}")

    def get_size_list(self, key: str, default: List[int]) -> List[int]:
        """Comma list of integers; an element may be an ``a..b`` range."""
        self._consumed.add(key)
        if key not in self._kv:
            return default
        out = []
        for raw in self._kv[key].split(","):
            tok = _trim(raw)
            try:
                dots = tok.find("..")
                if dots < 0:
                    out.append(parse_size(tok))
                else:
                    a, b = parse_size(_trim(tok[:dots])), parse_size(_trim(tok[dots + 2:]))
                    if b < a:
                        raise ValueError("descending range")
                    out.extend(range(a, b + 1))
            except ValueError:
                raise ConfigError(f"config key {key}: bad list element: {tok}") from None
        if not out:
            raise ConfigError(f"config key {key}: empty list")
        return out

    def get_double_list(self, key: str, default: List[float]) -> List[float]:
        self._consumed.add(key)
        if key not in self._kv:
            return default
        out = []
        for raw in self._kv[key].split(","):
            tok = _trim(raw)
            try:
                out.append(parse_double(tok))
            except ValueError:
                raise ConfigError(f"config key {key}: bad list element: {tok}") from None
        if not out:
            raise ConfigError(f"config key {key}: empty list")
        return out

    def get_string_list(self, key: str, default: List[str]) -> List[str]:
        self._consumed.add(key)
        if key not in self._kv:
            return default
        return [_trim(t) for t in self._kv[key].split(",")]

    def unconsumed(self) -> List[str]:
        return sorted(k for k in self._kv if k not in self._consumed)

    def reject_unknown(self) -> None:
        extra = self.unconsumed()
        if extra:
            raise ConfigError("unknown config keys: " + " ".join(extra))


def sweep_spec_from_config(cfg: Config) -> SweepSpec:
    """io.hpp:525-563: sweep.* for the grid, case.* for the shared settings;
    unknown keys are rejected."""
    spec = SweepSpec()
    spec.Lx = cfg.get_double_list("sweep.Lx", spec.Lx)
    spec.factors = cfg.get_size_list("sweep.factor", spec.factors)
    spec.ks = cfg.get_size_list("sweep.k", spec.ks)
    fams = []
    for s in cfg.get_string_list("sweep.family", [f.name for f in spec.families]):
        try:
            fams.append(family_from_string(s))
        except ValueError:
            raise ConfigError("config key sweep.family: unknown family " + s) from None
    spec.families = fams
    cycs = []
    for s in cfg.get_string_list("sweep.cycle", [c.name for c in spec.cycles]):
        try:
            cycs.append(cycle_from_string(s))
        except ValueError:
            raise ConfigError("config key sweep.cycle: unknown cycle " + s) from None
    spec.cycles = cycs
    b = spec.base
    b.n = cfg.get_size("case.n", b.n)
    try:
        b.driver = driver_from_string(cfg.get_string("case.driver", b.driver.name))
    except ValueError as e:
        raise ConfigError(f"config key case.driver: {e}") from None
    b.tol = cfg.get_double("case.tol", b.tol)
    b.restart = cfg.get_size("case.restart", b.restart)
    b.maxit = cfg.get_size("case.maxit", b.maxit)
    b.seeds.rhs = cfg.get_size("case.rhs_seed", b.seeds.rhs)
    b.seeds.eigen = cfg.get_size("case.eigen_seed", b.seeds.eigen)
    b.seeds.tuning = cfg.get_size("case.tuning_seed", b.seeds.tuning)
    b.lambda_max_multiplier = cfg.get_double("case.lambda_max_multiplier", b.lambda_max_multiplier)
    b.lambda_min_multiplier = cfg.get_double("case.lambda_min_multiplier", b.lambda_min_multiplier)
    b.eigen_iterations = cfg.get_size("case.eigen_iterations", b.eigen_iterations)
    b.estimate_c = cfg.get_bool("case.estimate_c", b.estimate_c)
    cfg.reject_unknown()
    return spec


__all__ = ["format_shortest", "parse_double", "parse_size", "KCSV_HEADER", "CsvOptions", "effective_lambda_min_mult",
           "csv_row", "write_csv_row", "write_csv", "CsvRow", "parse_csv", "write_beta_table_csv", "emit_sweep",
           "ConfigError", "Config", "sweep_spec_from_config"]
