"""BiCG / CGS / BiCGSTAB / GPBiCG on the B200 (drop-in for mpkrylov.solvers).

Same entry points, configuration and report as the reference
(/root/reference/pkg/src/mpkrylov/solvers.py:45-453): ``solve(A, b, cfg)``
and the per-method functions.  The whole solve -- binary64 ILU(0)
factorization, the method loop with its MC scalar recurrences and stopping
test, and the true residual -- runs on the GPU in one C-ABI call
(mpk_solve); the host only uploads A and b and downloads x.

Every combination the reference accepts runs on the device: precond
``ILU0_MIXED`` (the north-star configuration), ``ILU0_FULL`` and ``NONE``;
``spmv_mode`` "mixed" and "full", the latter with MC x MC products when the
matrix carries non-zero tail components (SURVEY.md section 8 a-f).

Extension over the reference report: ``history`` holds every norm2 value
the method computed (the reference's per-iteration residual norms, as
k-tuples), and ``factor_seconds`` / ``solve_seconds`` the device times.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .ilu import (
    IdentityPreconditioner,
    Ilu0Preconditioner,
    NumericBreakdownError,
    PrecondMode,
    SingularPivotError,
)
from .multicomponent import Precision
from .sparse import DenseVector, axpy, device_matrix, norm2

__all__ = [
    "SolverConfig",
    "SolveReport",
    "BreakdownError",
    "bicg",
    "cgs",
    "bicgstab",
    "gpbicg",
    "solve",
    "METHODS",
]

METHODS = ("bicg", "cgs", "bicgstab", "gpbicg")


class BreakdownError(ArithmeticError):
    pass


@dataclass
class SolverConfig:
    method: str = "bicg"
    precision: Precision = Precision.DD
    precond: PrecondMode = PrecondMode.NONE
    spmv_mode: str = "full"
    eps_rel: float = 1e-13
    eps_abs: float = 1e-100
    max_iter: int | None = None

    def __post_init__(self):
        if self.method not in METHODS:
            raise ValueError(f"unknown method {self.method!r}")
        if self.spmv_mode not in ("full", "mixed"):
            raise ValueError(f"unknown spmv mode {self.spmv_mode!r}")
        if self.eps_rel <= 0 or self.eps_abs <= 0:
            raise ValueError("eps_rel and eps_abs must be positive")
        if self.spmv_mode == "mixed" and self.precision.k < 2:
            raise ValueError("mixed SpMV needs a working precision above binary64")

    def resolved_max_iter(self, n: int) -> int:
        return 3 * n if self.max_iter is None else self.max_iter


@dataclass(eq=False)
class SolveReport:
    method: str
    precision: str
    precond: str
    spmv_mode: str
    iterations: int
    converged: bool
    total_seconds: float = 0.0
    ms_per_iteration: float = 0.0
    final_recursive_relres: float = float("nan")
    true_relres: float = float("nan")
    error_norm: float = float("nan")
    breakdown: str | None = None
    x: DenseVector | None = field(default=None, repr=False)
    history: list = field(default_factory=list, repr=False)
    factor_seconds: float = 0.0
    solve_seconds: float = 0.0


def _binary64_exact(A) -> bool:
    if A.precision.k == 1:
        return True
    ok = not np.any(A.val_re[:, 1:])
    if A.val_im is not None:
        ok = ok and not np.any(A.val_im[:, 1:])
    return bool(ok)


def _device_solve(A, b: DenseVector, cfg: SolverConfig, hist_cap: int | None = None):
    """One mpk_solve call; returns (MpkReport, x DenseVector|None, history)."""
    if A.n != b.n:
        raise ValueError("matrix/vector dimension mismatch")
    if A.field != b.field:
        raise ValueError(f"field mismatch: matrix {A.field}, vector {b.field}")
    if b.precision != cfg.precision:
        raise ValueError("vector precision must match cfg.precision")
    full = cfg.spmv_mode == "full"
    if full:
        # _Ctx.matvec -> spmv(A, v) (solvers.py:126-129, sparse.py:414-418): on
        # a binary64-valued matrix that IS the mixed computation bit for bit
        # (reference tests/test_sparse.py:130-147); an MC-valued matrix
        # multiplies with all its components (device_matrix attaches them)
        if A.precision.k != cfg.precision.k:
            raise ValueError("matrix and vector precision must match for spmv")
    elif not _binary64_exact(A):
        raise ValueError("mixed SpMV requires binary64-representable matrix values")
    k = cfg.precision.k
    n = A.n
    max_iter = cfg.resolved_max_iter(n)
    if hist_cap is None:
        hist_cap = 2 * max_iter + 2
    x = DenseVector.zeros(n, cfg.precision, A.field)
    hist = np.zeros((max(hist_cap, 1), k))
    rep = _lib.MpkReport()
    pre = {PrecondMode.NONE: 0, PrecondMode.ILU0_MIXED: 1, PrecondMode.ILU0_FULL: 2}[cfg.precond]
    with _lib.ctx_lock(_lib.context()):
        d = device_matrix(A)
        rc = _solve_locked(d, cfg, k, max_iter, b, x, hist, hist_cap, rep, pre, full)
    _lib.check(rc, "mpk_solve")
    h = [tuple(r) for r in hist[: min(rep.hist_len, hist_cap)]]
    return rep, (x if rep.has_x else None), h


def _solve_locked(d, cfg, k, max_iter, b, x, hist, hist_cap, rep, pre, full):
    with _lib.precond_scope(d.ctx, pre, spmv_full=full):
        rc = _lib.lib().mpk_solve(
            d.h, ctypes.c_int(_lib.METHOD_CODE[cfg.method]), ctypes.c_int(k),
            ctypes.c_double(cfg.eps_rel), ctypes.c_double(cfg.eps_abs),
            ctypes.c_int64(max_iter), _lib.dptr(_lib.f64(b.re)),
            _lib.dptr(None if b.im is None else _lib.f64(b.im)), _lib.dptr(x.re),
            _lib.dptr(x.im), _lib.dptr(hist), ctypes.c_int64(hist_cap), ctypes.byref(rep))
    return rc


def _breakdown_string(rep) -> str | None:
    code = rep.breakdown
    if code == 7:
        return f"SingularPivotError: {SingularPivotError(int(rep.bad_row), bool(rep.structural))}"
    if code == 8:
        return "NumericBreakdownError: non-finite value in ILU(0) factors"
    if code == 9:
        return "NumericBreakdownError: non-finite value in triangular sweep"
    return _lib.BREAKDOWN[code]


def solve(A, b: DenseVector, cfg: SolverConfig, x_star: DenseVector | None = None,
          parallel_spmv: bool = False) -> SolveReport:
    """Build the preconditioner, run the method, fill in the full report
    (solvers.py:418-453).  total_seconds includes the ILU(0) factorization."""
    t0 = time.perf_counter()
    rep, x, hist = _device_solve(A, b, cfg)
    elapsed = time.perf_counter() - t0
    out = SolveReport(
        method=cfg.method,
        precision=cfg.precision.label,
        precond=cfg.precond.value,
        spmv_mode=cfg.spmv_mode,
        iterations=int(rep.iterations),
        converged=bool(rep.converged),
        total_seconds=elapsed,
        breakdown=_breakdown_string(rep),
        x=x,
        history=hist,
        factor_seconds=rep.factor_ms * 1e-3,
        solve_seconds=rep.solve_ms * 1e-3,
    )
    if rep.breakdown in (7, 8, 9):
        return out
    if out.iterations > 0:
        out.ms_per_iteration = 1000.0 * elapsed / out.iterations
    out.final_recursive_relres = float(rep.final_recursive_relres)
    out.true_relres = float(rep.true_relres)
    if x is not None and x_star is not None:
        minus_one = -1.0
        out.error_norm = norm2(axpy(_unit(x, minus_one), x_star, x)).to_float()
    return out


def _unit(x: DenseVector, v: float):
    from .multicomponent import MCComplex, MCFloat

    r = MCFloat.from_float(v, x.precision)
    if x.field == "complex":
        return MCComplex(r, MCFloat.zero(x.precision))
    return r


def _method(name: str, A, b, cfg: SolverConfig, M=None) -> SolveReport:
    if M is None or isinstance(M, IdentityPreconditioner):  # M = I (reference default)
        pre = PrecondMode.NONE
    elif isinstance(M, Ilu0Preconditioner):
        pre = PrecondMode.ILU0_MIXED if M.mixed else PrecondMode.ILU0_FULL
    else:
        raise NotImplementedError(
            f"{name}(M=...) on the B200 path takes M=None or an ILU(0)-mixed "
            "preconditioner (build_preconditioner(A, PrecondMode.ILU0_MIXED))")
    c = SolverConfig(method=name, precision=cfg.precision, precond=pre,
                     spmv_mode=cfg.spmv_mode, eps_rel=cfg.eps_rel, eps_abs=cfg.eps_abs,
                     max_iter=cfg.max_iter)
    rep, x, hist = _device_solve(A, b, c)
    if rep.breakdown == 9:
        raise NumericBreakdownError("non-finite value in triangular sweep")
    return SolveReport(method=name, precision=cfg.precision.label,
                       precond=cfg.precond.value, spmv_mode=cfg.spmv_mode,
                       iterations=int(rep.iterations), converged=bool(rep.converged),
                       final_recursive_relres=float(rep.final_recursive_relres),
                       breakdown=_lib.BREAKDOWN[rep.breakdown], x=x, history=hist)


def bicg(A, b, cfg, M=None, parallel_spmv=False):
    """Two-sided preconditioned BiCG (solvers.py:183-226)."""
    return _method("bicg", A, b, cfg, M)


def cgs(A, b, cfg, M=None, parallel_spmv=False):
    """Preconditioned CGS (solvers.py:229-272)."""
    return _method("cgs", A, b, cfg, M)


def bicgstab(A, b, cfg, M=None, parallel_spmv=False):
    """Preconditioned BiCGSTAB (solvers.py:275-328)."""
    return _method("bicgstab", A, b, cfg, M)


def gpbicg(A, b, cfg, M=None, parallel_spmv=False):
    """GPBiCG on A M^-1 (solvers.py:331-412)."""
    return _method("gpbicg", A, b, cfg, M)
