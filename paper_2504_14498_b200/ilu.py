"""Binary64 ILU(0) on the B200 (drop-in for the mixed part of mpkrylov.ilu).

Reference: /root/reference/pkg/src/mpkrylov/ilu.py.  The factorization
(_factorize_tuples :178-276 with k=1) and the forward/backward sweeps
(:322-371) run as sync-free, one-row-per-thread CUDA kernels that keep the
reference's per-row operation order, so factors and sweep results are
bitwise identical (csrc/ilu.cu).  The working-precision ILU(0)
(PrecondMode.ILU0_FULL, ilu.py:279-281) runs in
K-component arithmetic on the device (csrc/ilu_mc.cu).
"""

from __future__ import annotations

import ctypes
from enum import Enum

import numpy as np

from . import _lib
from .multicomponent import Precision
from .sparse import CsrMatrix, DenseVector, device_matrix

__all__ = [
    "PrecondMode",
    "IluFactors",
    "SingularPivotError",
    "NumericBreakdownError",
    "ilu0_factorize",
    "ilu0_factorize_demoted",
    "ilu0_apply",
    "ilu0_apply_adjoint",
    "ilu0_apply_mixed",
    "ilu0_apply_adjoint_mixed",
    "IdentityPreconditioner",
    "Ilu0Preconditioner",
    "build_preconditioner",
]


class PrecondMode(Enum):
    NONE = "none"
    ILU0_FULL = "ilu0"
    ILU0_MIXED = "ilu0-mixed"

    @classmethod
    def from_label(cls, label: str) -> "PrecondMode":
        for m in cls:
            if m.value == label.lower():
                return m
        raise ValueError(f"unknown preconditioner mode {label!r}")


class SingularPivotError(ArithmeticError):
    """Zero or structurally missing pivot encountered at step k (ilu.py:60-66)."""

    def __init__(self, k: int, structural: bool = False):
        self.k = k
        kind = "structurally missing" if structural else "zero"
        super().__init__(f"ILU(0): {kind} pivot U[{k},{k}]")


class NumericBreakdownError(ArithmeticError):
    """Non-finite value produced during a triangular sweep (ilu.py:69-70)."""


class IluFactors:
    """Binary64 L/U values on A's pattern, resident on the device.

    ``val_re`` / ``val_im`` download the factors as (nnz, 1) arrays, like the
    reference's IluFactors for k = 1 (ilu.py:89-110)."""

    def __init__(self, A, dev):
        self.n = int(A.n)
        self.row_ptr = A.row_ptr
        self.col_idx = A.col_idx
        self.diag_ptr = getattr(A, "diag_ptr", None)
        self.precision = Precision.F64
        self._dev = dev
        self._cx = A.val_im is not None
        self._host = None

    @property
    def field(self) -> str:
        return "complex" if self._cx else "real"

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def _download(self):
        if self._host is None:
            re = np.zeros(self.nnz)
            im = np.zeros(self.nnz) if self._cx else None
            _lib.check(_lib.lib().mpk_ilu0_download(self._dev.h, _lib.dptr(re),
                                                    _lib.dptr(im)), "download")
            self._host = (re, im)
        return self._host

    @property
    def val_re(self) -> np.ndarray:
        return self._download()[0][:, None]

    @property
    def val_im(self):
        im = self._download()[1]
        return None if im is None else im[:, None]


def _factor(A) -> IluFactors:
    if A.val_im is not None or A.val_re is not None:
        pass
    d = device_matrix(A)
    bad = ctypes.c_int64(-1)
    st = ctypes.c_int32(0)
    rc = _lib.lib().mpk_ilu0_factor(d.h, ctypes.byref(bad), ctypes.byref(st))
    if rc == _lib.MPK_SINGULAR_PIVOT:
        raise SingularPivotError(int(bad.value), structural=bool(st.value))
    _lib.check(rc, "mpk_ilu0_factor")
    d.factored = True
    return IluFactors(A, d)


def ilu0_factorize_demoted(A) -> IluFactors:
    """Demote values to binary64, then factorize in binary64 (ilu.py:284-286)."""
    return _factor(A.demoted() if A.precision.k > 1 else A)


class IluFactorsMC(IluFactors):
    """Working-precision factors (k = 2..4) resident on the device
    (csrc/ilu_mc.cu); ``val_re`` / ``val_im`` download them as (nnz, k).  The device
    matrix keeps one such set (the latest k factorised)."""

    def __init__(self, A, dev, precision):
        super().__init__(A, dev)
        self.precision = precision

    def _download(self):
        if self._host is None:
            k = self.precision.k
            lu = np.zeros((self.nnz, 2 * k if self._cx else k))
            _lib.check(_lib.lib().mpk_ilu0_download_full(self._dev.h, ctypes.c_int(k),
                                                         _lib.dptr(lu)), "download_full")
            self._host = (np.ascontiguousarray(lu[:, :k]),
                          np.ascontiguousarray(lu[:, k:]) if self._cx else None)
        return self._host

    @property
    def val_re(self) -> np.ndarray:
        return self._download()[0]

    @property
    def val_im(self):
        return self._download()[1]


def ilu0_factorize(A) -> IluFactors:
    """Zero-fill ILU at the matrix's working precision (ilu.py:279-281): k = 1
    binary64, k = 2..4 in K-component arithmetic with the reference's fused
    a - b*c; an MC-valued matrix is factored with all its components
    (device_matrix attaches them)."""
    if A.precision.k == 1:
        return _factor(A)
    d = device_matrix(A)
    bad = ctypes.c_int64(-1)
    st = ctypes.c_int32(0)
    rc = _lib.lib().mpk_ilu0_factor_full(d.h, ctypes.c_int(A.precision.k), ctypes.byref(bad),
                                         ctypes.byref(st))
    if rc == _lib.MPK_SINGULAR_PIVOT:
        raise SingularPivotError(int(bad.value), structural=bool(st.value))
    _lib.check(rc, "mpk_ilu0_factor_full")
    return IluFactorsMC(A, d, A.precision)


def _check_apply(F: IluFactors, r: DenseVector):
    if F.n != r.n:
        raise ValueError(f"dimension mismatch: factors n={F.n}, vector n={r.n}")
    if F.field != r.field:
        raise ValueError(f"field mismatch: factors {F.field}, vector {r.field}")


def _apply_f64(F: IluFactors, r: DenseVector, adjoint: bool) -> DenseVector:
    _check_apply(F, r)
    if r.precision.k != 1:
        raise ValueError("factor precision must match the vector precision")
    z_re = np.zeros(F.n)
    z_im = np.zeros(F.n) if F._cx else None
    rr = _lib.f64(r.re[:, 0])
    ri = None if r.im is None else _lib.f64(r.im[:, 0])
    rc = _lib.lib().mpk_ilu0_apply_f64(F._dev.h, _lib.dptr(rr), _lib.dptr(ri),
                                       _lib.dptr(z_re), _lib.dptr(z_im),
                                       ctypes.c_int(int(adjoint)))
    _lib.check(rc, "mpk_ilu0_apply_f64")
    return DenseVector(z_re[:, None].copy(), None if z_im is None else z_im[:, None].copy(),
                       Precision.F64)


def _apply_full(F, r: DenseVector, adjoint: bool) -> DenseVector:
    _check_apply(F, r)
    if F.precision != r.precision:
        raise ValueError("factor precision must match the vector precision")
    k = F.precision.k
    cx = F._cx
    rin = np.concatenate([r.re, r.im]) if cx else r.re
    z = np.zeros((2 * F.n if cx else F.n, k))
    rc = _lib.lib().mpk_ilu0_apply_full_ex(F._dev.h, ctypes.c_int(k), _lib.dptr(_lib.f64(rin)),
                                           _lib.dptr(z), ctypes.c_int(int(adjoint)))
    if rc == _lib.MPK_NUMERIC_BREAKDOWN:
        raise NumericBreakdownError("non-finite value in triangular sweep")
    _lib.check(rc, "mpk_ilu0_apply_full_ex")
    if cx:
        return DenseVector(z[:F.n].copy(), z[F.n:].copy(), F.precision)
    return DenseVector(z, None, F.precision)


def ilu0_apply(F: IluFactors, r: DenseVector) -> DenseVector:
    """z = U^-1 (L^-1 r) at the factors' precision (ilu.py:410-420)."""
    if isinstance(F, IluFactorsMC):
        return _apply_full(F, r, False)
    return _apply_f64(F, r, False)


def ilu0_apply_adjoint(F: IluFactors, r: DenseVector) -> DenseVector:
    """z = (LU)^-H r (ilu.py:423-433)."""
    if isinstance(F, IluFactorsMC):
        return _apply_full(F, r, True)
    return _apply_f64(F, r, True)


def _apply_mixed(F: IluFactors, r: DenseVector, adjoint: bool) -> DenseVector:
    if r.precision.k < 2:
        raise ValueError("mixed apply expects a working precision above binary64")
    if F.n != r.n or F.field != r.field:
        raise ValueError("factors/vector mismatch")
    k = r.precision.k
    z = DenseVector.zeros(r.n, r.precision, r.field)
    rc = _lib.lib().mpk_ilu0_apply_mixed(
        F._dev.h, ctypes.c_int(k), _lib.dptr(_lib.f64(r.re)),
        _lib.dptr(None if r.im is None else _lib.f64(r.im)), _lib.dptr(z.re),
        _lib.dptr(z.im), ctypes.c_int(int(adjoint)))
    _lib.check(rc, "mpk_ilu0_apply_mixed")
    return z


def ilu0_apply_mixed(F64: IluFactors, r: DenseVector) -> DenseVector:
    """promote . binary64 apply . demote (ilu.py:448-458)."""
    return _apply_mixed(F64, r, False)


def ilu0_apply_adjoint_mixed(F64: IluFactors, r: DenseVector) -> DenseVector:
    return _apply_mixed(F64, r, True)


class IdentityPreconditioner:
    """No-op preconditioner (ilu.py:478-491)."""

    mode = PrecondMode.NONE

    def apply(self, r: DenseVector) -> DenseVector:
        return r

    def apply_adjoint(self, r: DenseVector) -> DenseVector:
        return r

    @property
    def setup_seconds(self) -> float:
        return 0.0


class Ilu0Preconditioner:
    """ILU(0)-mixed preconditioner object (ilu.py:494-511)."""

    def __init__(self, factors: IluFactors, mixed: bool, setup_seconds: float = 0.0):
        self.factors = factors
        self.mixed = mixed
        self.mode = PrecondMode.ILU0_MIXED if mixed else PrecondMode.ILU0_FULL
        self.setup_seconds = setup_seconds

    def apply(self, r: DenseVector) -> DenseVector:
        if self.mixed and r.precision.k > 1:
            return ilu0_apply_mixed(self.factors, r)
        return ilu0_apply(self.factors, r)

    def apply_adjoint(self, r: DenseVector) -> DenseVector:
        if self.mixed and r.precision.k > 1:
            return ilu0_apply_adjoint_mixed(self.factors, r)
        return ilu0_apply_adjoint(self.factors, r)


def build_preconditioner(A, mode: PrecondMode):
    """ilu.py:514-522."""
    if mode == PrecondMode.NONE:
        return IdentityPreconditioner()
    if mode == PrecondMode.ILU0_FULL:
        return Ilu0Preconditioner(ilu0_factorize(A), mixed=False)
    if mode == PrecondMode.ILU0_MIXED:
        return Ilu0Preconditioner(ilu0_factorize_demoted(A), mixed=True)
    raise ValueError(f"unsupported preconditioner mode {mode}")
