"""ctypes binding of the C oracle (see oracle/__init__.py: test-only)."""

from __future__ import annotations

import ctypes
import os
import pathlib
import subprocess

import numpy as np

__all__ = [
    "lib",
    "build",
    "OrcReport",
    "BREAKDOWN",
    "METHOD_CODE",
    "mc_op",
    "renorm",
    "spmv_mixed",
    "hdot",
    "norm2",
    "axpy",
    "ilu0_factor",
    "ilu0_apply_f64",
    "ilu0_apply_mixed",
    "solve",
    "solve_batch",
    "set_threads",
]

_DIR = pathlib.Path(__file__).resolve().parent
_SO = _DIR / "liborc.so"
_lib = None

BREAKDOWN = {
    0: None,
    1: "sigma_zero",
    2: "rho_zero",
    3: "omega_zero",
    4: "nonfinite_residual",
    5: "breakdown_ls",
    6: "zeta_zero",
    7: "SingularPivotError",
    8: "NumericBreakdownError",
    9: "NumericBreakdownError",
}
METHOD_CODE = {"bicg": 0, "cgs": 1, "bicgstab": 2, "gpbicg": 3}


class OrcReport(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int64),
        ("converged", ctypes.c_int32),
        ("breakdown", ctypes.c_int32),
        ("bad_row", ctypes.c_int64),
        ("structural", ctypes.c_int32),
        ("has_x", ctypes.c_int32),
        ("final_recursive_relres", ctypes.c_double),
        ("true_relres", ctypes.c_double),
        ("hist_len", ctypes.c_int64),
        ("factor_seconds", ctypes.c_double),
        ("loop_seconds", ctypes.c_double),
    ]


def build(force: bool = False) -> pathlib.Path:
    src = _DIR / "mpk_oracle.c"
    if force or not _SO.exists() or _SO.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_DIR)], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not _SO.exists():
            build()
        _lib = ctypes.CDLL(str(_SO))
        _lib.orc_solve.restype = ctypes.c_int
        _lib.orc_renorm.restype = None
    return _lib


def _p(a):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _pi(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def set_threads(t: int) -> None:
    lib().orc_set_threads(ctypes.c_int(int(t)))


def mc_op(op: str, a, b=None, ai=None, bi=None):
    """Element-wise MC op on (n,k) arrays: add sub mul div sqrt cmul cdiv."""
    L = lib()
    a = _f(a)
    n, k = a.shape
    out = np.zeros((n, k))
    if op in ("add", "sub", "mul", "div"):
        b = _f(b)
        fn = {"add": L.orc_add, "sub": L.orc_sub, "mul": L.orc_mul,
              "div": L.orc_div}[op]
        for i in range(n):
            fn(_p(a[i]), _p(b[i]), _p(out[i]), ctypes.c_int(k))
        return out
    if op == "sqrt":
        for i in range(n):
            L.orc_sqrt(_p(a[i]), _p(out[i]), ctypes.c_int(k))
        return out
    if op in ("cmul", "cdiv"):
        b, ai, bi = _f(b), _f(ai), _f(bi)
        oi = np.zeros((n, k))
        fn = L.orc_cx_mul if op == "cmul" else L.orc_cx_div
        for i in range(n):
            fn(_p(a[i]), _p(ai[i]), _p(b[i]), _p(bi[i]), _p(out[i]), _p(oi[i]),
               ctypes.c_int(k))
        return out, oi
    raise ValueError(op)


def renorm(terms, k: int):
    terms = _f(terms)
    n, m = terms.shape
    out = np.zeros((n, k))
    lib().orc_ew_renorm(ctypes.c_int64(n), ctypes.c_int(m), _p(terms), _p(out),
                        ctypes.c_int(k))
    return out


def spmv_mixed(n, rp, ci, vre, vim, x_re, x_im=None, adjoint=False):
    rp, ci = _i(rp), _i(ci)
    vre = _f(vre)
    vim = None if vim is None else _f(vim)
    x_re = _f(x_re)
    k = x_re.shape[1]
    y_re = np.zeros_like(x_re)
    y_im = None
    if vim is not None:
        x_im = _f(x_im)
        y_im = np.zeros_like(x_re)
    fn = lib().orc_spmv_adjoint_mixed if adjoint else lib().orc_spmv_mixed
    fn(ctypes.c_int64(n), _pi(rp), _pi(ci), _p(vre), _p(vim), ctypes.c_int(k),
       _p(x_re), _p(x_im), _p(y_re), _p(y_im))
    return y_re, y_im


def hdot(x_re, y_re, x_im=None, y_im=None):
    x_re, y_re = _f(x_re), _f(y_re)
    n, k = x_re.shape
    o_re = np.zeros(k)
    o_im = np.zeros(k) if x_im is not None else None
    lib().orc_hdot(ctypes.c_int64(n), ctypes.c_int(k), _p(x_re),
                   _p(None if x_im is None else _f(x_im)), _p(y_re),
                   _p(None if y_im is None else _f(y_im)), _p(o_re), _p(o_im))
    return o_re, o_im


def norm2(x_re, x_im=None):
    x_re = _f(x_re)
    n, k = x_re.shape
    out = np.zeros(k)
    lib().orc_norm2(ctypes.c_int64(n), ctypes.c_int(k), _p(x_re),
                    _p(None if x_im is None else _f(x_im)), _p(out))
    return out


def axpy(a_re, x_re, y_re, a_im=None, x_im=None, y_im=None):
    x_re, y_re = _f(x_re), _f(y_re)
    n, k = x_re.shape
    a = np.zeros(4)
    a[:k] = a_re
    ai = None
    if a_im is not None:
        ai = np.zeros(4)
        ai[:k] = a_im
    o_re = np.zeros_like(x_re)
    o_im = np.zeros_like(x_re) if x_im is not None else None
    lib().orc_axpy(ctypes.c_int64(n), ctypes.c_int(k), _p(a), _p(ai), _p(x_re),
                   _p(None if x_im is None else _f(x_im)), _p(y_re),
                   _p(None if y_im is None else _f(y_im)), _p(o_re), _p(o_im))
    return o_re, o_im


def _diag_ptr(n, rp, ci):
    dp = np.full(n, -1, dtype=np.int64)
    for i in range(n):
        lo, hi = rp[i], rp[i + 1]
        pos = np.searchsorted(ci[lo:hi], i)
        if pos < hi - lo and ci[lo + pos] == i:
            dp[i] = lo + pos
    return dp


def ilu0_factor(n, rp, ci, vre, vim=None):
    """Returns (status, lu_re, lu_im, bad_row, structural)."""
    rp, ci = _i(rp), _i(ci)
    dp = _diag_ptr(n, rp, ci)
    vre = _f(vre)
    vim = None if vim is None else _f(vim)
    lu_re = np.zeros_like(vre)
    lu_im = None if vim is None else np.zeros_like(vim)
    bad = ctypes.c_int64(-1)
    st = ctypes.c_int(0)
    rc = lib().orc_ilu0_factor(ctypes.c_int64(n), _pi(rp), _pi(ci), _pi(dp),
                               _p(vre), _p(vim), _p(lu_re), _p(lu_im),
                               ctypes.byref(bad), ctypes.byref(st))
    return rc, lu_re, lu_im, bad.value, st.value


def ilu0_apply_f64(n, rp, ci, lu_re, lu_im, r_re, r_im=None, adjoint=False):
    rp, ci = _i(rp), _i(ci)
    dp = _diag_ptr(n, rp, ci)
    r_re = _f(r_re)
    z_re = np.zeros(n)
    z_im = None
    if lu_im is not None:
        r_im = _f(r_im)
        z_im = np.zeros(n)
    rc = lib().orc_ilu0_apply_f64(ctypes.c_int64(n), _pi(rp), _pi(ci), _pi(dp),
                                  _p(_f(lu_re)),
                                  _p(None if lu_im is None else _f(lu_im)),
                                  _p(r_re), _p(r_im), _p(z_re), _p(z_im),
                                  ctypes.c_int(1 if adjoint else 0))
    return rc, z_re, z_im


def ilu0_apply_mixed(n, rp, ci, lu_re, lu_im, r_re, r_im=None, adjoint=False):
    """promote . f64 apply . demote (ilu.py:448-470) on (n,k) arrays."""
    k = r_re.shape[1]
    if lu_im is None:
        rc, z, _ = ilu0_apply_f64(n, rp, ci, lu_re, None, r_re[:, 0].copy(),
                                  adjoint=adjoint)
        out = np.zeros((n, k))
        out[:, 0] = z
        return rc, out, None
    c = r_re[:, 0] + 1j * r_im[:, 0]
    rc, zr, zi = ilu0_apply_f64(n, rp, ci, lu_re, lu_im, c.real.copy(),
                                c.imag.copy(), adjoint=adjoint)
    zc = zr + 1j * zi
    o_re = np.zeros((n, k))
    o_im = np.zeros((n, k))
    o_re[:, 0] = zc.real
    o_im[:, 0] = zc.imag
    return rc, o_re, o_im


def solve(n, rp, ci, vre, vim, method, k, b_re, b_im=None, eps_rel=1e-13,
          eps_abs=1e-100, max_iter=None, precond_ilu=True, hist_cap=None):
    """Run solvers.solve() semantics; returns (report, x_re, x_im, hist)."""
    rp, ci = _i(rp), _i(ci)
    vre = _f(vre)
    vim = None if vim is None else _f(vim)
    b_re = _f(b_re)
    b_im = None if b_im is None else _f(b_im)
    if max_iter is None:
        max_iter = 3 * n
    if hist_cap is None:
        hist_cap = 2 * max_iter + 4
    x_re = np.zeros((n, k))
    x_im = np.zeros((n, k)) if vim is not None else None
    hist = np.zeros((hist_cap, k))
    rep = OrcReport()
    lib().orc_solve(ctypes.c_int64(n), _pi(rp), _pi(ci), _p(vre), _p(vim),
                    ctypes.c_int(METHOD_CODE[method]), ctypes.c_int(k),
                    ctypes.c_double(eps_rel), ctypes.c_double(eps_abs),
                    ctypes.c_int64(max_iter), ctypes.c_int(1 if precond_ilu else 0),
                    _p(b_re), _p(b_im), _p(x_re), _p(x_im), _p(hist),
                    ctypes.c_int64(hist_cap), ctypes.byref(rep))
    return rep, x_re, x_im, hist[: min(rep.hist_len, hist_cap)]


def solve_batch(systems, method, k, eps_rel, eps_abs, max_iter, threads):
    """systems: list of (n, rp, ci, vre, b_re); returns reports, xs."""
    ns = len(systems)
    keep = []
    N = (ctypes.c_int64 * ns)()
    RP = (ctypes.POINTER(ctypes.c_int64) * ns)()
    CI = (ctypes.POINTER(ctypes.c_int64) * ns)()
    AV = (ctypes.POINTER(ctypes.c_double) * ns)()
    B = (ctypes.POINTER(ctypes.c_double) * ns)()
    X = (ctypes.POINTER(ctypes.c_double) * ns)()
    xs = []
    for s, (n, rp, ci, vre, b) in enumerate(systems):
        rp, ci, vre, b = _i(rp), _i(ci), _f(vre), _f(b)
        x = np.zeros((n, k))
        keep += [rp, ci, vre, b]
        xs.append(x)
        N[s] = n
        RP[s] = _pi(rp)
        CI[s] = _pi(ci)
        AV[s] = _p(vre)
        B[s] = _p(b)
        X[s] = _p(x)
    reps = (OrcReport * ns)()
    lib().orc_solve_batch(ctypes.c_int(ns), N, RP, CI, AV,
                          ctypes.c_int(METHOD_CODE[method]), ctypes.c_int(k),
                          ctypes.c_double(eps_rel), ctypes.c_double(eps_abs),
                          ctypes.c_int64(max_iter), B, X, reps,
                          ctypes.c_int(threads))
    return list(reps), xs


os.environ.setdefault("MPK_ORACLE", str(_SO))
