"""ctypes binding of the B200 hot-path library (include/mpk_b200.h).

The product path has NO CPU fallback: if libmpkb200.so is missing, or no
CUDA device is present, the device entry points raise.  Only the host-side
MC scalar arithmetic (mpk_mc_host, used by MCFloat/MCComplex) works without
a GPU, exactly like the reference's scalar types run on the host.
"""

from __future__ import annotations

import ctypes
import pathlib
import threading

import numpy as np

import os

# MPK_B200_LIB: another build of the same library (A/B measurements of kernel variants)
_SO = pathlib.Path(os.environ.get("MPK_B200_LIB") or
                   pathlib.Path(__file__).resolve().parent / "_lib" / "libmpkb200.so")
_lib = None
_lock = threading.RLock()  # re-entrant: context() loads the library under it
_ctx = {}

MPK_OK = 0
MPK_SINGULAR_PIVOT = 1
MPK_NUMERIC_BREAKDOWN = 2
MPK_INVALID = 3
MPK_CUDA_ERROR = 4

METHOD_CODE = {"bicg": 0, "cgs": 1, "bicgstab": 2, "gpbicg": 3}
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

# every symbol include/mpk_b200.h declares (checked by tests/test_host.py)
EXPORTS = (
    "mpk_last_error", "mpk_version", "mpk_ctx_create", "mpk_ctx_destroy",
    "mpk_ctx_synchronize", "mpk_csr_upload", "mpk_csr_free", "mpk_ilu0_factor",
    "mpk_ilu0_download", "mpk_ilu0_apply_f64", "mpk_ilu0_apply_mixed",
    "mpk_spmv_mixed", "mpk_hdot", "mpk_norm2", "mpk_axpy", "mpk_mc_elementwise",
    "mpk_mc_host", "mpk_solve", "mpk_plane_ld", "mpk_solve_dev", "mpk_to_planar",
    "mpk_from_planar", "mpk_solve_batch", "mpk_ctx_stream", "mpk_bench_apply", "mpk_bench_spmv", "mpk_sweep_info",
    "mpk_csr_set_values", "mpk_csr_set_mc_values", "mpk_spmv_full", "mpk_run_jobs",
    "mpk_ctx_set_option", "mpk_thread_set_option",
    "mpk_comm_unique_id", "mpk_comm_create", "mpk_comm_create_local", "mpk_comm_destroy",
    "mpk_comm_rank", "mpk_comm_world", "mpk_solve_dev_sharded",
    "mpk_ilu0_factor_full", "mpk_ilu0_download_full", "mpk_ilu0_apply_full",
    "mpk_ilu0_apply_full_ex",
)

MPK_OPT_REDUCTION = 1
REDUCTION_MODE = {"tree": 0, "sequential": 1}
MPK_OPT_PRECOND = 2  # 0: none (M = I), 1: ILU(0)-mixed (default)
MPK_OPT_SPMV = 3  # per-thread: 0 mixed, 1 full (the matrix's attached MC values)


class precond_scope:
    """Selects the preconditioner of the calling thread's solves for one call
    (MPK_OPT_PRECOND: 0 none, 1 ILU(0)-mixed, 2 working-precision ILU(0))
    through the library's thread-local override, so concurrent solves on one
    context never see each other's setting; cleared on exit."""

    def __init__(self, ctx, ilu, spmv_full: bool = False):
        # ilu: True -> 1 (default), False -> 0, or the option value itself
        self.ctx = ctx
        self.value = int(ilu)
        self.spmv_full = bool(spmv_full)

    def __enter__(self):
        check(lib().mpk_thread_set_option(ctypes.c_int(MPK_OPT_PRECOND),
                                          ctypes.c_int64(self.value)),
              "mpk_thread_set_option")
        if self.spmv_full:
            check(lib().mpk_thread_set_option(ctypes.c_int(MPK_OPT_SPMV), ctypes.c_int64(1)),
                  "mpk_thread_set_option")
        return self

    def __exit__(self, *exc):
        lib().mpk_thread_set_option(ctypes.c_int(MPK_OPT_PRECOND), ctypes.c_int64(-1))
        lib().mpk_thread_set_option(ctypes.c_int(MPK_OPT_SPMV), ctypes.c_int64(0))
        return False


class MpkReport(ctypes.Structure):
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
        ("factor_ms", ctypes.c_double),
        ("solve_ms", ctypes.c_double),
        ("total_ms", ctypes.c_double),
        ("launches", ctypes.c_int64),
    ]


class MpkJob(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_void_p),
        ("method", ctypes.c_int32),
        ("k", ctypes.c_int32),
        ("eps_rel", ctypes.c_double),
        ("eps_abs", ctypes.c_double),
        ("max_iter", ctypes.c_int64),
        ("b_re", ctypes.c_void_p),
        ("b_im", ctypes.c_void_p),
        ("x_re", ctypes.c_void_p),
        ("x_im", ctypes.c_void_p),
        ("val_re", ctypes.c_void_p),
        ("val_im", ctypes.c_void_p),
        ("hist", ctypes.c_void_p),
        ("hist_cap", ctypes.c_int64),
        ("rep", MpkReport),
        ("rc", ctypes.c_int32),
    ]


class ExtensionMissing(RuntimeError):
    pass


def lib():
    """Load libmpkb200.so (fails loudly when it was not built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not _SO.exists():
                    raise ExtensionMissing(
                        f"{_SO} not built: run `python -c 'import __graft_entry__ as g;"
                        f" g.build()'` (nvcc, sm_100a)")
                L = ctypes.CDLL(str(_SO))
                L.mpk_last_error.restype = ctypes.c_char_p
                L.mpk_plane_ld.restype = ctypes.c_int64
                L.mpk_plane_ld.argtypes = [ctypes.c_int64]
                _lib = L
    return _lib


def last_error() -> str:
    return lib().mpk_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    if rc == MPK_OK:
        return
    msg = last_error()
    if rc == MPK_INVALID:
        raise ValueError(msg)
    if rc == MPK_NUMERIC_BREAKDOWN:
        from .ilu import NumericBreakdownError

        raise NumericBreakdownError(msg)
    if rc == MPK_SINGULAR_PIVOT:
        raise RuntimeError(msg)  # callers translate with the row index
    raise RuntimeError(f"CUDA error in {what}: {msg}")


def context(device: int = 0):
    """Per-device context (one CUDA stream), created on first use."""
    c = _ctx.get(device)
    if c is None:
        with _lock:
            c = _ctx.get(device)
            if c is None:
                p = ctypes.c_void_p()
                check(lib().mpk_ctx_create(ctypes.c_int(device), ctypes.byref(p)),
                      "mpk_ctx_create")
                c = p
                _ctx[device] = c
    return c


_ctx_locks: dict = {}


def ctx_lock(ctx) -> "threading.RLock":
    """One lock per device context: a context is one CUDA stream plus cached
    solver plans (captured graphs), so calls on it from several host threads
    take turns.  Contexts are independent of each other (mpk_run_jobs runs
    one native thread per context concurrently)."""
    key = ctx.value if hasattr(ctx, "value") else int(ctx)
    lk = _ctx_locks.get(key)
    if lk is None:
        with _lock:
            lk = _ctx_locks.setdefault(key, threading.RLock())
    return lk


def dptr(a):
    """Pointer argument for an array (or None).  The returned object holds a
    reference to `a` (numpy's data_as), so a temporary such as the
    contiguous copy `f64(v[:, 0])` stays alive until the call returns."""
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.c_void_p)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def plane_ld(n: int) -> int:
    return int(lib().mpk_plane_ld(ctypes.c_int64(n)))


def set_reduction(mode: str, device: int = 0) -> None:
    """Reduction order of hdot/norm2 and of the solvers' dot products:
    "tree" (default, fixed-shape parallel tree) or "sequential" (the
    reference's ascending accumulation, _kernels.py:487-552 -- bit-identical
    to it, one dependent chain of n MC additions per reduction)."""
    if mode not in REDUCTION_MODE:
        raise ValueError(f"unknown reduction mode {mode!r} (tree | sequential)")
    check(lib().mpk_ctx_set_option(context(device), ctypes.c_int(MPK_OPT_REDUCTION),
                                   ctypes.c_int64(REDUCTION_MODE[mode])),
          "mpk_ctx_set_option")


class reduction_mode:
    """Context manager: `with reduction_mode("sequential"): ...`"""

    def __init__(self, mode: str, device: int = 0):
        self.mode, self.device = mode, device

    def __enter__(self):
        set_reduction(self.mode, self.device)
        return self

    def __exit__(self, *exc):
        set_reduction("tree", self.device)
        return False
