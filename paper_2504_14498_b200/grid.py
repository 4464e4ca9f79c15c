"""Benchmark grid and report emission: the paper's
Tables 1/2/4 layout over the device path.

Same schema and entry points as the reference harness (bench.py:44-309):
``build_problem`` (x* = sqrt(2)*[1..n] real, sqrt(2+3i)*[1..n] complex, in
the working precision; b = A x* by full SpMV), ``default_grid`` (every
method x DD/TD/QD x {plain, ILU(0), mixed SpMV, mixed SpMV + ILU(0)_d}),
``run_benchmark`` -> ``BenchRow`` list (a failing cell becomes a
non-converged row), ``emit_report`` (CSV with the reference header, or JSON;
optional Table-4 ratio section), ``parse_report`` (CSV round trip) and
``ratio_rows`` (per-iteration time ratios ILU(0)/plain, ILU(0)_d/plain_d,
ILU(0)/ILU(0)_d).  Every cell is a device solve (solvers.solve); the device
path covers binary64-valued matrices, where spmv_mode 'full' and 'mixed' are
the same computation bit for bit.
"""

from __future__ import annotations

import csv
import ctypes
import io
import json
from dataclasses import asdict, dataclass

import numpy as np

from . import _lib
from .ilu import PrecondMode
from .mmio import coo_to_csr, read_matrix_market
from .multicomponent import MCComplex, MCFloat, Precision
from .solvers import SolveReport, SolverConfig, solve
from .sparse import DenseVector, spmv

__all__ = ["CSV_HEADER", "ProblemSpec", "BenchRow", "RatioRow", "build_problem",
           "load_matrix", "default_grid", "run_cell", "run_benchmark", "emit_report",
           "parse_report", "ratio_rows"]

CSV_HEADER = ["matrix", "method", "precision", "precond", "spmv_mode", "iterations",
              "converged", "total_s", "ms_per_iter", "true_relres", "err2"]
RATIO_HEADER = ["matrix", "method", "precision", "ilu0_over_plain", "ilu0d_over_plaind",
                "ilu0_over_ilu0d"]


@dataclass
class ProblemSpec:
    matrix_name: str
    field: str
    n: int
    x_star: DenseVector
    b: DenseVector


@dataclass
class BenchRow:
    matrix: str
    method: str
    precision: str
    precond: str
    spmv_mode: str
    iterations: int
    converged: bool
    total_s: float
    ms_per_iter: float
    true_relres: float
    err2: float


@dataclass
class RatioRow:
    matrix: str
    method: str
    precision: str
    ilu0_over_plain: float
    ilu0d_over_plaind: float
    ilu0_over_ilu0d: float


def _scale_dev(alpha, x: DenseVector) -> DenseVector:
    """alpha * x element-wise on the device in the reference's operand order
    (scale_real / scale_cx, _kernels.py:437-464: mul(alpha, x_i))."""
    k, n = x.precision.k, x.n
    cx = x.field == "complex"
    ar = np.tile(np.asarray(alpha.re.components if cx else alpha.components, np.float64), (n, 1))
    ai = np.tile(np.asarray(alpha.im.components, np.float64), (n, 1)) if cx else None
    o = np.zeros((n, k))
    oi = np.zeros((n, k)) if cx else None
    rc = _lib.lib().mpk_mc_elementwise(
        _lib.context(), ctypes.c_int(5 if cx else 2), ctypes.c_int(k), ctypes.c_int64(n),
        _lib.dptr(ar), _lib.dptr(ai), _lib.dptr(_lib.f64(x.re)),
        _lib.dptr(None if x.im is None else _lib.f64(x.im)), _lib.dptr(o), _lib.dptr(oi))
    _lib.check(rc, "mpk_mc_elementwise")
    return DenseVector(o, oi, x.precision)


def build_problem(A, precision: Precision, matrix_name: str = "") -> ProblemSpec:
    """x* = sqrt(2)*[1..n] (complex: sqrt(2+3i)*[1..n]) at the working
    precision and b = A x* (bench.py:86-102)."""
    if A.precision != precision:
        raise ValueError("load the matrix at the requested precision first")
    n = A.n
    ramp = np.arange(1, n + 1, dtype=np.float64)
    if A.field == "real":
        x_ramp = DenseVector.from_float64(ramp, precision)
        root = MCFloat.from_float(2.0, precision).sqrt()
    else:
        x_ramp = DenseVector.from_float64(ramp.astype(np.complex128), precision)
        root = MCComplex.from_complex(2 + 3j, precision).sqrt()
    x_star = _scale_dev(root, x_ramp)
    return ProblemSpec(matrix_name, A.field, n, x_star, spmv(A, x_star))


def load_matrix(path, precision: Precision):
    return coo_to_csr(read_matrix_market(path), precision)


def default_grid(methods=None, precisions=None):
    """(method, precision, precond, spmv_mode) cells of the paper grid."""
    methods = list(methods) if methods else ["bicg", "cgs", "bicgstab", "gpbicg"]
    precisions = list(precisions) if precisions else [Precision.DD, Precision.TD, Precision.QD]
    variants = ((PrecondMode.NONE, "full"), (PrecondMode.ILU0_FULL, "full"),
                (PrecondMode.NONE, "mixed"), (PrecondMode.ILU0_MIXED, "mixed"))
    return [(m, p, pre, mode) for m in methods for p in precisions
            for pre, mode in variants if not (mode == "mixed" and p.k < 2)]


def _row(name: str, rep: SolveReport) -> BenchRow:
    return BenchRow(name, rep.method, rep.precision, rep.precond, rep.spmv_mode,
                    int(rep.iterations), bool(rep.converged), float(rep.total_seconds),
                    float(rep.ms_per_iteration), float(rep.true_relres),
                    float(rep.error_norm))


def run_cell(A, problem: ProblemSpec, cfg: SolverConfig,
             parallel_spmv: bool = False) -> BenchRow:
    """One cell (bench.py:172-176).  `parallel_spmv` asks the reference for
    its row-parallel CPU SpMV; the device SpMV is row-parallel already and
    computes the same rows, so the flag changes nothing here."""
    return _row(problem.matrix_name,
                solve(A, problem.b, cfg, x_star=problem.x_star, parallel_spmv=parallel_spmv))


def run_benchmark(suite, jobs: int = 1, log=None) -> list:
    """Cells (A, problem, cfg); a failing cell becomes a non-converged row
    with NaN timings (bench.py:179-216).  jobs = 1 runs them one after
    another (uncontended timings); jobs > 1 hands them to a pool of `jobs`
    threads -- solves that share a device context queue behind each other on
    its stream, so, as in the reference, the timing fields are then
    unreliable while every other field is unchanged."""
    if not callable(log) and log is not None:
        raise TypeError("log must be a callable taking one string (or None)")

    def one(cell):
        A, problem, cfg = cell
        try:
            row = run_cell(A, problem, cfg)
        except Exception as exc:  # reported in the row, the grid continues
            nan = float("nan")
            row = BenchRow(problem.matrix_name, cfg.method, cfg.precision.label,
                           cfg.precond.value, cfg.spmv_mode, 0, False, nan, nan, nan, nan)
            if log:
                log(f"cell failed: {cfg.method}/{cfg.precision.label}: {exc}")
        if log:
            log(f"{row.matrix} {row.method} {row.precision} {row.precond} {row.spmv_mode}: "
                f"iters={row.iterations} converged={row.converged} total={row.total_s:.3f}s")
        return row

    suite = list(suite)
    if int(jobs) > 1:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=int(jobs)) as pool:
            return list(pool.map(one, suite))
    return [one(cell) for cell in suite]


def ratio_rows(rows) -> list:
    """Table-4 per-iteration time ratios for every (matrix, method, precision)."""
    by = {(r.matrix, r.method, r.precision, r.precond, r.spmv_mode): r for r in rows}

    def q(a, b):
        if a is None or b is None or not b.ms_per_iter:
            return float("nan")
        return a.ms_per_iter / b.ms_per_iter

    out, seen = [], set()
    for r in rows:
        key = (r.matrix, r.method, r.precision)
        if key in seen:
            continue
        seen.add(key)
        plain, ilu = by.get(key + ("none", "full")), by.get(key + ("ilu0", "full"))
        plain_d, ilu_d = by.get(key + ("none", "mixed")), by.get(key + ("ilu0-mixed", "mixed"))
        if ilu is None and ilu_d is None:
            continue
        out.append(RatioRow(*key, q(ilu, plain), q(ilu_d, plain_d), q(ilu, ilu_d)))
    return out


def emit_report(rows, fmt: str = "csv", out=None, ratios: bool = False) -> str:
    if not rows:
        raise ValueError("no rows to report")
    if fmt == "csv":
        buf = io.StringIO()
        w = csv.writer(buf, lineterminator="\n")
        w.writerow(CSV_HEADER)
        for r in rows:
            w.writerow([r.matrix, r.method, r.precision, r.precond, r.spmv_mode, r.iterations,
                        r.converged, repr(r.total_s), repr(r.ms_per_iter),
                        repr(r.true_relres), repr(r.err2)])
        if ratios:
            w.writerow([])
            w.writerow(RATIO_HEADER)
            for rr in ratio_rows(rows):
                w.writerow([rr.matrix, rr.method, rr.precision, repr(rr.ilu0_over_plain),
                            repr(rr.ilu0d_over_plaind), repr(rr.ilu0_over_ilu0d)])
        text = buf.getvalue()
    elif fmt == "json":
        payload = {"rows": [asdict(r) for r in rows]}
        if ratios:
            payload["ratios"] = [asdict(rr) for rr in ratio_rows(rows)]
        text = json.dumps(payload, indent=2)
    else:
        raise ValueError(f"unknown report format {fmt!r}")
    if out is not None:
        out.write(text)
    return text


def parse_report(text: str) -> list:
    """The CSV main table back into rows (round trip of emit_report)."""
    rd = csv.reader(io.StringIO(text))
    if next(rd) != CSV_HEADER:
        raise ValueError("unexpected CSV header")
    rows = []
    for rec in rd:
        if not rec:
            break  # ratio section
        rows.append(BenchRow(rec[0], rec[1], rec[2], rec[3], rec[4], int(rec[5]),
                             rec[6] == "True", float(rec[7]), float(rec[8]), float(rec[9]),
                             float(rec[10])))
    return rows
