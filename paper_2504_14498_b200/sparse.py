"""CSR matrices, MC vectors and the hot-path vector kernels on the B200.

Drop-in for the hot-path part of mpkrylov.sparse
(/root/reference/pkg/src/mpkrylov/sparse.py:192-604): the container types
keep the reference's host layouts ((n,k) float64 component arrays, int64
CSR), and every kernel runs on the GPU through the C ABI
(include/mpk_b200.h) with the reference's exact per-element operation
sequences.  Reductions (hdot/norm2) use a fixed-shape device tree (see
DESIGN.md); SpMV / axpy results are bitwise equal to the reference.
"""

from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import _lib
from .multicomponent import MCComplex, MCFloat, Precision

__all__ = [
    "CsrMatrix",
    "DenseVector",
    "spmv",
    "spmv_adjoint",
    "spmv_mixed",
    "spmv_adjoint_mixed",
    "hdot",
    "dot",
    "norm2",
    "axpy",
    "scale",
    "vec_sub",
    "vec_add",
    "vec_copy",
    "device_matrix",
]


class CsrMatrix:
    """Square CSR matrix with multi-component values (sparse.py:192-272)."""

    def __init__(self, n, row_ptr, col_idx, val_re, val_im, precision: Precision):
        self.n = int(n)
        self.row_ptr = row_ptr
        self.col_idx = col_idx
        self.val_re = val_re
        self.val_im = val_im
        self.precision = precision
        self._validate()
        self.diag_ptr = self._find_diagonals()

    @property
    def field(self) -> str:
        return "real" if self.val_im is None else "complex"

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def _validate(self):
        n = self.n
        rp, ci = np.asarray(self.row_ptr), np.asarray(self.col_idx)
        if len(rp) != n + 1 or rp[0] != 0 or rp[-1] != len(ci):
            raise ValueError("inconsistent CSR row_ptr")
        if np.any(np.diff(rp) < 0):
            raise ValueError("row_ptr must be non-decreasing")
        k = self.precision.k
        if self.val_re.shape != (len(ci), k):
            raise ValueError("val_re shape mismatch")
        if self.val_im is not None and self.val_im.shape != (len(ci), k):
            raise ValueError("val_im shape mismatch")
        if len(ci):
            row_of = np.repeat(np.arange(n), np.diff(rp))
            bad = (ci < 0) | (ci >= n)
            same_row = np.diff(row_of) == 0
            bad[1:] |= same_row & (np.diff(ci) <= 0)
            if np.any(bad):
                i = int(row_of[np.argmax(bad)])
                raise ValueError(f"row {i}: columns must be strictly increasing and in range")

    def _find_diagonals(self):
        n = self.n
        rp, ci = np.asarray(self.row_ptr), np.asarray(self.col_idx)
        dp = np.full(n, -1, dtype=np.int64)
        if len(ci):
            row_of = np.repeat(np.arange(n), np.diff(rp))
            hit = np.nonzero(ci == row_of)[0]
            dp[row_of[hit]] = hit
        return dp

    def demoted(self) -> "CsrMatrix":
        vre = np.ascontiguousarray(self.val_re[:, :1])
        vim = None if self.val_im is None else np.ascontiguousarray(self.val_im[:, :1])
        return CsrMatrix(self.n, self.row_ptr, self.col_idx, vre, vim, Precision.F64)

    def promoted(self, target: Precision) -> "CsrMatrix":
        if self.precision.k > target.k:
            raise ValueError("use demoted() to narrow")
        vre = np.zeros((self.nnz, target.k))
        vre[:, : self.precision.k] = self.val_re
        vim = None
        if self.val_im is not None:
            vim = np.zeros((self.nnz, target.k))
            vim[:, : self.precision.k] = self.val_im
        return CsrMatrix(self.n, self.row_ptr, self.col_idx, vre, vim, target)

    @classmethod
    def from_binary64(cls, n, row_ptr, col_idx, val_re, val_im=None,
                      precision: Precision = Precision.F64) -> "CsrMatrix":
        """Exactly promoted matrix from binary64 arrays (helper)."""
        nnz = len(col_idx)
        vre = np.zeros((nnz, precision.k))
        vre[:, 0] = val_re
        vim = None
        if val_im is not None:
            vim = np.zeros((nnz, precision.k))
            vim[:, 0] = val_im
        return cls(n, np.asarray(row_ptr, np.int64), np.asarray(col_idx, np.int64),
                   vre, vim, precision)


class DenseVector:
    """Length-n vector of multi-component scalars (sparse.py:341-404)."""

    __slots__ = ("re", "im", "precision")

    def __init__(self, re: np.ndarray, im: np.ndarray | None, precision: Precision):
        if re.ndim != 2 or re.shape[1] != precision.k:
            raise ValueError("component array must be (n, k)")
        if im is not None and im.shape != re.shape:
            raise ValueError("re/im shape mismatch")
        self.re = re
        self.im = im
        self.precision = precision

    @property
    def n(self) -> int:
        return self.re.shape[0]

    @property
    def field(self) -> str:
        return "real" if self.im is None else "complex"

    @classmethod
    def zeros(cls, n: int, precision: Precision, field: str = "real") -> "DenseVector":
        re = np.zeros((n, precision.k))
        im = np.zeros((n, precision.k)) if field == "complex" else None
        return cls(re, im, precision)

    @classmethod
    def from_float64(cls, values, precision: Precision) -> "DenseVector":
        values = np.asarray(values)
        n = len(values)
        re = np.zeros((n, precision.k))
        if np.iscomplexobj(values):
            im = np.zeros((n, precision.k))
            re[:, 0] = values.real
            im[:, 0] = values.imag
            return cls(re, im, precision)
        re[:, 0] = values.astype(np.float64)
        return cls(re, None, precision)

    def copy(self) -> "DenseVector":
        return DenseVector(self.re.copy(), None if self.im is None else self.im.copy(),
                           self.precision)

    def demote_to_float64(self) -> np.ndarray:
        if self.im is None:
            return self.re[:, 0].copy()
        return self.re[:, 0] + 1j * self.im[:, 0]

    def get(self, i: int):
        if self.im is None:
            return MCFloat(tuple(self.re[i]))
        return MCComplex(MCFloat(tuple(self.re[i])), MCFloat(tuple(self.im[i])))

    def set(self, i: int, value):
        if self.im is None:
            self.re[i] = value.components
        else:
            self.re[i] = value.re.components
            self.im[i] = value.im.components


# ---------------------------------------------------------------------
# device matrix handles (one upload per matrix object)
# ---------------------------------------------------------------------
def _words(a):
    return np.ascontiguousarray(a).view(np.uint64).ravel()


def _fingerprint(*arrays):
    """Content fingerprint of host arrays: the wrapping sum of the raw 64-bit
    words (any change of a single word changes it; one streaming pass) plus
    the xor of every 61st word, so that compensating multi-word changes are
    unlikely to go unnoticed either."""
    out = []
    for a in arrays:
        if a is None:
            out.append(None)
            continue
        w = _words(np.asarray(a))
        if not w.size:
            out.append((0, 0, 0))
            continue
        out.append((w.size, int(w.sum(dtype=np.uint64)), int(np.bitwise_xor.reduce(w[::61]))))
    return tuple(out)


class _DevMatrix:
    """Device copy of one CsrMatrix: the binary64 (demoted) values every
    kernel of the mixed path reads and, for an MC-valued matrix (non-zero
    tail components), all k components for spmv_mode 'full' and the
    working-precision ILU(0).  `sync` re-uploads values the caller changed in
    place since the last call (the reference reads A afresh on every call)."""

    def __init__(self, A, device: int = 0):
        L = _lib.lib()
        self.ctx = _lib.context(device)
        self.n = int(A.n)
        rp = _lib.i64(A.row_ptr)
        ci = _lib.i64(A.col_idx)
        vre = _lib.f64(np.asarray(A.val_re)[:, 0])
        vim = None if A.val_im is None else _lib.f64(np.asarray(A.val_im)[:, 0])
        h = ctypes.c_void_p()
        _lib.check(L.mpk_csr_upload(self.ctx, ctypes.c_int64(self.n),
                                    ctypes.c_int64(len(ci)), _lib.dptr(rp), _lib.dptr(ci),
                                    _lib.dptr(vre), _lib.dptr(vim), ctypes.byref(h)),
                   "mpk_csr_upload")
        self.h = h
        self.cx = vim is not None
        self.factored = False
        self.mc_k = 0
        self.pattern = _fingerprint(A.row_ptr, A.col_idx)
        self.values = None
        self._fin = weakref.finalize(self, L.mpk_csr_free, h)
        self.sync(A, heads_current=True)

    def sync(self, A, heads_current: bool = False) -> None:
        fp = _fingerprint(A.val_re, A.val_im)
        if fp == self.values:
            return
        L = _lib.lib()
        vre_all = np.asarray(A.val_re)
        vim_all = None if A.val_im is None else np.asarray(A.val_im)
        if not heads_current:
            # the head columns are strided views: keep their contiguous copies
            # alive in locals for the duration of the call
            hre = _lib.f64(vre_all[:, 0])
            him = None if vim_all is None else _lib.f64(vim_all[:, 0])
            _lib.check(L.mpk_csr_set_values(self.h, _lib.dptr(hre), _lib.dptr(him)),
                       "mpk_csr_set_values")
            self.factored = False
        k = vre_all.shape[1]
        tails = k > 1 and (bool(np.any(vre_all[:, 1:])) or
                           (vim_all is not None and bool(np.any(vim_all[:, 1:]))))
        if tails:
            fre = _lib.f64(vre_all)
            fim = None if vim_all is None else _lib.f64(vim_all)
            _lib.check(L.mpk_csr_set_mc_values(self.h, ctypes.c_int(k), _lib.dptr(fre),
                                               _lib.dptr(fim)), "mpk_csr_set_mc_values")
            self.mc_k = k
        elif self.mc_k:
            _lib.check(L.mpk_csr_set_mc_values(self.h, ctypes.c_int(0), None, None),
                       "mpk_csr_set_mc_values")
            self.mc_k = 0
        self.values = fp


_dev_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def device_matrix(A) -> _DevMatrix:
    """The device copy of A, cached per matrix object and kept in step with
    in-place changes of A's values (fingerprint check per call) or pattern
    (fresh upload).  Works for this package's CsrMatrix and the reference's."""
    try:
        d = _dev_cache.get(A)
    except TypeError:
        d = None
    if d is not None and d.pattern != _fingerprint(A.row_ptr, A.col_idx):
        d = None
    if d is None:
        d = _DevMatrix(A)
        try:
            _dev_cache[A] = d
        except TypeError:
            pass
    else:
        d.sync(A)
    return d


def _check_pair(A, x: DenseVector):
    if A.n != x.n:
        raise ValueError(f"dimension mismatch: matrix n={A.n}, vector n={x.n}")
    if A.field != x.field:
        raise ValueError(f"field mismatch: matrix {A.field}, vector {x.field}")


def _check_mixed(A64, x: DenseVector):
    _check_pair(A64, x)
    if A64.precision.k != 1:
        raise ValueError("mixed SpMV requires a binary64 matrix (use demoted())")
    if x.precision.k < 2:
        raise ValueError("mixed SpMV requires a working precision above binary64")


def _spmv_dev(A, x: DenseVector, adjoint: bool) -> DenseVector:
    d = device_matrix(A)
    k = x.precision.k
    out = DenseVector.zeros(A.n, x.precision, A.field)
    xr, xi = _lib.f64(x.re), None if x.im is None else _lib.f64(x.im)
    _lib.check(_lib.lib().mpk_spmv_mixed(d.h, ctypes.c_int(k), _lib.dptr(xr),
                                         _lib.dptr(xi), _lib.dptr(out.re),
                                         _lib.dptr(out.im), ctypes.c_int(int(adjoint))),
               "mpk_spmv_mixed")
    return out


def spmv_mixed(A64, x: DenseVector) -> DenseVector:
    """y = A x with binary64 entries promoted exactly (sparse.py:465-480)."""
    _check_mixed(A64, x)
    return _spmv_dev(A64, x, False)


def spmv_adjoint_mixed(A64, x: DenseVector) -> DenseVector:
    """y = A^H x (sparse.py:483-496), gather over the transpose in the
    reference's ascending-source-row order."""
    _check_mixed(A64, x)
    return _spmv_dev(A64, x, True)


def _spmv_full_dev(A, x: DenseVector, adjoint: bool, what: str) -> DenseVector:
    _check_pair(A, x)
    if A.precision.k != x.precision.k:
        raise ValueError(f"matrix and vector precision must match for {what}")
    d = device_matrix(A)
    k = x.precision.k
    out = DenseVector.zeros(A.n, x.precision, A.field)
    xr, xi = _lib.f64(x.re), None if x.im is None else _lib.f64(x.im)
    _lib.check(_lib.lib().mpk_spmv_full(d.h, ctypes.c_int(k), _lib.dptr(xr), _lib.dptr(xi),
                                        _lib.dptr(out.re), _lib.dptr(out.im),
                                        ctypes.c_int(int(adjoint))), "mpk_spmv_full")
    return out


def spmv(A, x: DenseVector, parallel: bool = False) -> DenseVector:
    """y = A x with products and accumulation at the value precision
    (sparse.py:414-435 -> _kernels.py:224-240 / 300-323): MC x MC products
    for an MC-valued matrix; for a binary64-valued one the mixed kernel,
    which is the same computation bit for bit (tests/test_sparse.py:130-147).
    `parallel` selects the reference's row-parallel CPU variant, which
    computes the same rows; the device kernel is row-parallel already."""
    return _spmv_full_dev(A, x, False, "spmv")


def spmv_adjoint(A, x: DenseVector) -> DenseVector:
    """y = A^H x (sparse.py:438-451 -> _kernels.py:266-278 / 356-376), as a
    gather over the transposed pattern in the reference's scatter order
    (ascending source row per output row), entries conjugated."""
    return _spmv_full_dev(A, x, True, "spmv_adjoint")


def _check_vecs(x: DenseVector, y: DenseVector):
    if x.n != y.n or x.field != y.field or x.precision != y.precision:
        raise ValueError("vector length/field/precision mismatch")


def hdot(x: DenseVector, y: DenseVector):
    """sum conj(x_i) y_i (sparse.py:509-517), fixed-shape device tree."""
    _check_vecs(x, y)
    k = x.precision.k
    o_re = np.zeros(k)
    o_im = np.zeros(k) if x.im is not None else None
    _lib.check(_lib.lib().mpk_hdot(
        _lib.context(), ctypes.c_int64(x.n), ctypes.c_int(k), _lib.dptr(_lib.f64(x.re)),
        _lib.dptr(None if x.im is None else _lib.f64(x.im)), _lib.dptr(_lib.f64(y.re)),
        _lib.dptr(None if y.im is None else _lib.f64(y.im)), _lib.dptr(o_re),
        _lib.dptr(o_im)), "mpk_hdot")
    if x.im is None:
        return MCFloat(tuple(o_re))
    return MCComplex(MCFloat(tuple(o_re)), MCFloat(tuple(o_im)))


def dot(x: DenseVector, y: DenseVector):
    """Unconjugated sum (sparse.py:520-529)."""
    if x.field == "real":
        return hdot(x, y)
    return hdot(DenseVector(x.re, -x.im, x.precision), y)


def norm2(x: DenseVector) -> MCFloat:
    k = x.precision.k
    out = np.zeros(k)
    _lib.check(_lib.lib().mpk_norm2(
        _lib.context(), ctypes.c_int64(x.n), ctypes.c_int(k), _lib.dptr(_lib.f64(x.re)),
        _lib.dptr(None if x.im is None else _lib.f64(x.im)), _lib.dptr(out)),
        "mpk_norm2")
    return MCFloat(tuple(out))


def axpy(alpha, x: DenseVector, y: DenseVector) -> DenseVector:
    """y + alpha x (sparse.py:542-560), bitwise equal to the reference."""
    _check_vecs(x, y)
    k = x.precision.k
    out = DenseVector.zeros(x.n, x.precision, x.field)
    a = np.zeros(4)
    ai = None
    if isinstance(alpha, MCComplex):
        a[:k] = alpha.re.components
        ai = np.zeros(4)
        ai[:k] = alpha.im.components
    elif isinstance(alpha, MCFloat):
        a[:k] = alpha.components
    else:
        a[:k] = alpha
    if x.im is not None and ai is None:
        ai = np.zeros(4)
    _lib.check(_lib.lib().mpk_axpy(
        _lib.context(), ctypes.c_int64(x.n), ctypes.c_int(k), _lib.dptr(a),
        _lib.dptr(ai), _lib.dptr(_lib.f64(x.re)),
        _lib.dptr(None if x.im is None else _lib.f64(x.im)), _lib.dptr(_lib.f64(y.re)),
        _lib.dptr(None if y.im is None else _lib.f64(y.im)), _lib.dptr(out.re),
        _lib.dptr(out.im)), "mpk_axpy")
    return out


def _elementwise(op: int, k: int, a_re, a_im, b_re, b_im, cx: bool):
    n = len(b_re)
    o_re = np.zeros((n, k))
    o_im = np.zeros((n, k)) if cx else None
    ins = [None if a is None else _lib.f64(a) for a in (a_re, a_im, b_re, b_im)]  # kept alive
    _lib.check(_lib.lib().mpk_mc_elementwise(
        _lib.context(), ctypes.c_int(op), ctypes.c_int(k), ctypes.c_int64(n),
        _lib.dptr(ins[0]), _lib.dptr(ins[1]), _lib.dptr(ins[2]), _lib.dptr(ins[3]),
        _lib.dptr(o_re), _lib.dptr(o_im)), "mpk_mc_elementwise")
    return o_re, o_im


def scale(alpha, x: DenseVector) -> DenseVector:
    """alpha * x (sparse.py:563-579 -> _kernels.py scale_real / scale_cx:
    alpha is the left factor of every product)."""
    k = x.precision.k
    ar = np.zeros((x.n, k))
    if x.im is None:
        ar[:] = alpha.components if isinstance(alpha, MCFloat) else alpha
        o_re, _ = _elementwise(2, k, ar, None, x.re, None, False)
        return DenseVector(o_re, None, x.precision)
    ai = np.zeros((x.n, k))
    if isinstance(alpha, MCComplex):
        ar[:] = alpha.re.components
        ai[:] = alpha.im.components
    else:
        ar[:] = alpha.components if isinstance(alpha, MCFloat) else alpha
    o_re, o_im = _elementwise(5, k, ar, ai, x.re, x.im, True)
    return DenseVector(o_re, o_im, x.precision)


def _planes(op: int, x: DenseVector, y: DenseVector) -> DenseVector:
    _check_vecs(x, y)
    k = x.precision.k
    o_re, _ = _elementwise(op, k, x.re, None, y.re, None, False)
    o_im = None
    if x.im is not None:
        o_im, _ = _elementwise(op, k, x.im, None, y.im, None, False)
    return DenseVector(o_re, o_im, x.precision)


def vec_sub(x: DenseVector, y: DenseVector) -> DenseVector:
    """x - y (sparse.py:582-590), real and imaginary planes separately."""
    return _planes(1, x, y)


def vec_add(x: DenseVector, y: DenseVector) -> DenseVector:
    """x + y (sparse.py:593-600)."""
    return _planes(0, x, y)


def vec_copy(x: DenseVector) -> DenseVector:
    return x.copy()
