"""Generate golden vectors from the REFERENCE implementation (run here only).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Imports the read-only reference package from /root/reference/pkg/src and
records, on seeded inputs, the outputs of the functions on the hot path:
MC scalar ops (_mccore.py), mixed SpMV / adjoint / hdot / norm2 / axpy
(sparse.py), binary64 ILU(0) factors and applies (ilu.py), and full
solver runs (solvers.py) with their per-iteration residual-norm history
(captured by wrapping mpkrylov.solvers.norm2 during the method call,
SURVEY.md section 4.4).  The reference is not available on the GPU box, so
the .npz files written next to this script are committed and the tests
compare the oracle and the device path against them.
"""

from __future__ import annotations

import os
import pathlib
import sys
import time

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import mpkrylov  # noqa: E402
from mpkrylov import _mccore, ilu, solvers, sparse  # noqa: E402
from mpkrylov.multicomponent import Precision  # noqa: E402

from paper_2504_14498_b200 import problems  # noqa: E402

PREC = {2: Precision.DD, 3: Precision.TD, 4: Precision.QD}
LABEL = {"dd": 2, "td": 3, "qd": 4}


def rand_mc(rng, k, scale=1.0):
    """Random renormalized k-tuple with content in every limb (the
    reference's own test helper recipe, tests/conftest.py:42-45)."""
    terms = [rng.uniform(-1.0, 1.0) * scale * 2.0 ** (-52 * i) for i in range(k)]
    return _mccore.renormalize(terms, k)


def batch(rng, k, n, spread=True):
    return np.array([rand_mc(rng, k, 10.0 ** rng.integers(-6, 7) if spread else 1.0)
                     for _ in range(n)])


def special_mc(k):
    """Edge operands: zeros, signed zeros, exact ones, zero tails, ties."""
    z = [0.0] * k
    out = [tuple(z), tuple([-0.0] * k), tuple([1.0] + z[1:]),
           tuple([-1.0] + z[1:]), tuple([3.0] + z[1:]),
           tuple([1e-300] + z[1:]), tuple([2.0 ** 60] + z[1:])]
    if k >= 2:
        out.append(tuple([1.0, 2.0 ** -60] + z[2:]))
        out.append(tuple([1.0, -(2.0 ** -53)] + z[2:]))
    return np.array(out)


# ---------------------------------------------------------------------
def gen_mc_ops():
    data = {}
    for k in (2, 3, 4):
        rng = np.random.default_rng(100 + k)
        a = np.concatenate([batch(rng, k, 400), special_mc(k)])
        b = np.concatenate([batch(rng, k, 400), special_mc(k)[::-1]])
        # cross the specials with randoms
        sp = special_mc(k)
        a = np.concatenate([a, np.repeat(sp, 3, axis=0)])
        b = np.concatenate([b, batch(rng, k, 3 * len(sp))])
        data[f"k{k}_a"] = a
        data[f"k{k}_b"] = b
        data[f"k{k}_add"] = np.array([_mccore.mc_add(tuple(x), tuple(y)) for x, y in zip(a, b)])
        data[f"k{k}_sub"] = np.array([_mccore.mc_sub(tuple(x), tuple(y)) for x, y in zip(a, b)])
        data[f"k{k}_mul"] = np.array([_mccore.mc_mul(tuple(x), tuple(y)) for x, y in zip(a, b)])
        nz = [i for i in range(len(b)) if b[i][0] != 0.0]
        data[f"k{k}_div_idx"] = np.array(nz)
        data[f"k{k}_div"] = np.array([_mccore.mc_div(tuple(a[i]), tuple(b[i])) for i in nz])
        pos = np.abs(a)
        pos = np.array([_mccore.renormalize(list(r), k) for r in pos])
        data[f"k{k}_sqrt_in"] = pos
        data[f"k{k}_sqrt"] = np.array([_mccore.mc_sqrt(tuple(x)) for x in pos])
        raw = rng.uniform(-1, 1, size=(500, 7)) * 10.0 ** rng.integers(-8, 9, size=(500, 7))
        raw[::7, 3] = 0.0
        raw[::11, 0] = -0.0
        data[f"k{k}_renorm_in"] = raw
        data[f"k{k}_renorm"] = np.array([_mccore.renorm_terms(list(r), k) for r in raw])
        # complex
        ar, ai, br, bi = (batch(rng, k, 200, spread=False) for _ in range(4))
        cm = [_mccore.cx_mul((tuple(ar[i]), tuple(ai[i])), (tuple(br[i]), tuple(bi[i])))
              for i in range(200)]
        cd = [_mccore.cx_div((tuple(ar[i]), tuple(ai[i])), (tuple(br[i]), tuple(bi[i])))
              for i in range(200)]
        for nm, v in (("ar", ar), ("ai", ai), ("br", br), ("bi", bi)):
            data[f"k{k}_c{nm}"] = v
        data[f"k{k}_cmul_re"] = np.array([c[0] for c in cm])
        data[f"k{k}_cmul_im"] = np.array([c[1] for c in cm])
        data[f"k{k}_cdiv_re"] = np.array([c[0] for c in cd])
        data[f"k{k}_cdiv_im"] = np.array([c[1] for c in cd])
        # promoted-binary64 products (SpMV/axpy specialisations)
        f = rng.standard_normal(300) * 10.0 ** rng.integers(-5, 6, size=300)
        x = batch(rng, k, 300)
        data[f"k{k}_f"] = f
        data[f"k{k}_x"] = x
        zt = lambda v: (float(v),) + (0.0,) * (k - 1)  # noqa: E731
        data[f"k{k}_mul_lf"] = np.array([_mccore.mc_mul(zt(f[i]), tuple(x[i])) for i in range(300)])
        data[f"k{k}_mul_rf"] = np.array([_mccore.mc_mul(tuple(x[i]), zt(f[i])) for i in range(300)])
        g = rng.standard_normal(300)
        data[f"k{k}_g"] = g
        data[f"k{k}_mul_ff"] = np.array([_mccore.mc_mul(zt(f[i]), zt(g[i])) for i in range(300)])
    np.savez_compressed(HERE / "mc_ops.npz", **data)


def random_dd(rng, n, density, complex_field=False):
    """Diagonally dominant random sparse matrix (tests/conftest.py:58-80)."""
    mask = rng.random((n, n)) < density
    np.fill_diagonal(mask, True)
    if complex_field:
        vals = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
    else:
        vals = rng.uniform(-1, 1, (n, n)).astype(complex)
    vals = vals * mask
    for i in range(n):
        vals[i, i] = np.abs(vals[i]).sum() + 1.0
    rows, cols = np.nonzero(mask)
    vre = vals[rows, cols].real.astype(float)
    vim = vals[rows, cols].imag.astype(float) if complex_field else None
    coo = sparse.CooMatrix(n, n, rows.astype(np.int64), cols.astype(np.int64),
                           vre, vim, "general")
    return sparse.coo_to_csr(coo, Precision.F64)


def mc_vec(rng, n, k, cx):
    re = np.array([rand_mc(rng, k) for _ in range(n)])
    im = np.array([rand_mc(rng, k) for _ in range(n)]) if cx else None
    return sparse.DenseVector(re, im, PREC[k])


def gen_sparse():
    data = {}
    for cx in (False, True):
        tag = "c" if cx else "r"
        rng = np.random.default_rng(14 if not cx else 15)
        A64 = random_dd(rng, 50, 0.15, cx)
        data[f"{tag}_rp"] = A64.row_ptr
        data[f"{tag}_ci"] = A64.col_idx
        data[f"{tag}_vre"] = A64.val_re[:, 0]
        if cx:
            data[f"{tag}_vim"] = A64.val_im[:, 0]
        for k in (2, 3, 4):
            x = mc_vec(rng, 50, k, cx)
            y = mc_vec(rng, 50, k, cx)
            data[f"{tag}{k}_xre"] = x.re
            data[f"{tag}{k}_yre"] = y.re
            if cx:
                data[f"{tag}{k}_xim"] = x.im
                data[f"{tag}{k}_yim"] = y.im
            s = sparse.spmv_mixed(A64, x)
            sa = sparse.spmv_adjoint_mixed(A64, x)
            data[f"{tag}{k}_spmv_re"] = s.re
            data[f"{tag}{k}_adj_re"] = sa.re
            if cx:
                data[f"{tag}{k}_spmv_im"] = s.im
                data[f"{tag}{k}_adj_im"] = sa.im
            # promoted binary64 input (the M^-1-output case)
            xf = sparse.DenseVector.from_float64(x.demote_to_float64(), PREC[k])
            sf = sparse.spmv_mixed(A64, xf)
            data[f"{tag}{k}_spmvf_re"] = sf.re
            if cx:
                data[f"{tag}{k}_spmvf_im"] = sf.im
            h = sparse.hdot(x, y)
            nr = sparse.norm2(x)
            data[f"{tag}{k}_norm2"] = np.array(nr.components)
            if cx:
                data[f"{tag}{k}_hdot_re"] = np.array(h.re.components)
                data[f"{tag}{k}_hdot_im"] = np.array(h.im.components)
                al = mpkrylov.MCComplex(mpkrylov.MCFloat(rand_mc(rng, k)),
                                        mpkrylov.MCFloat(rand_mc(rng, k)))
                data[f"{tag}{k}_alpha_re"] = np.array(al.re.components)
                data[f"{tag}{k}_alpha_im"] = np.array(al.im.components)
            else:
                data[f"{tag}{k}_hdot_re"] = np.array(h.components)
                al = mpkrylov.MCFloat(rand_mc(rng, k))
                data[f"{tag}{k}_alpha_re"] = np.array(al.components)
            ax = sparse.axpy(al, x, y)
            data[f"{tag}{k}_axpy_re"] = ax.re
            if cx:
                data[f"{tag}{k}_axpy_im"] = ax.im
    np.savez_compressed(HERE / "sparse_small.npz", **data)


def _factor_record(data, tag, A64, rng):
    F = ilu.ilu0_factorize_demoted(A64)
    data[f"{tag}_rp"] = A64.row_ptr
    data[f"{tag}_ci"] = A64.col_idx
    data[f"{tag}_vre"] = A64.val_re[:, 0]
    data[f"{tag}_lu_re"] = F.val_re[:, 0]
    cx = A64.field == "complex"
    if cx:
        data[f"{tag}_vim"] = A64.val_im[:, 0]
        data[f"{tag}_lu_im"] = F.val_im[:, 0]
    n = A64.n
    for k in (2, 4):
        r = mc_vec(rng, n, k, cx)
        z = ilu.ilu0_apply_mixed(F, r)
        za = ilu.ilu0_apply_adjoint_mixed(F, r)
        data[f"{tag}_k{k}_r_re"] = r.re
        data[f"{tag}_k{k}_z_re"] = z.re
        data[f"{tag}_k{k}_za_re"] = za.re
        if cx:
            data[f"{tag}_k{k}_r_im"] = r.im
            data[f"{tag}_k{k}_z_im"] = z.im
            data[f"{tag}_k{k}_za_im"] = za.im


def gen_ilu():
    data = {}
    rng = np.random.default_rng(21)
    # SPEC.md:267-268 tridiagonal example
    coo = sparse.CooMatrix(3, 3, np.array([0, 0, 1, 1, 1, 2, 2], dtype=np.int64),
                           np.array([0, 1, 0, 1, 2, 1, 2], dtype=np.int64),
                           np.array([2.0, -1, -1, 2, -1, -1, 2]), None, "general")
    _factor_record(data, "tri3", sparse.coo_to_csr(coo, Precision.F64), rng)
    _factor_record(data, "rnd_r", random_dd(rng, 40, 0.2), rng)
    _factor_record(data, "rnd_c", random_dd(rng, 40, 0.2, True), rng)
    p = problems.cfg1()
    A64 = sparse.CsrMatrix(p.n, p.row_ptr, p.col_idx, p.val_re[:, None], None, Precision.F64)
    _factor_record(data, "cfg1", A64, rng)
    # a matrix whose ILU(0) hits a zero pivot at row 2, and one missing a diagonal
    coo = sparse.CooMatrix(3, 3, np.array([0, 0, 1, 1, 2, 2], dtype=np.int64),
                           np.array([0, 1, 0, 1, 1, 2], dtype=np.int64),
                           np.array([1.0, 1.0, 1.0, 1.0, 1.0, 1.0]), None, "general")
    Az = sparse.coo_to_csr(coo, Precision.F64)
    try:
        ilu.ilu0_factorize_demoted(Az)
        data["zero_pivot_row"] = np.array(-1)
    except ilu.SingularPivotError as e:
        data["zero_pivot_row"] = np.array(e.k)
        data["zero_pivot_msg"] = np.array(str(e))
    data["zp_rp"], data["zp_ci"], data["zp_vre"] = Az.row_ptr, Az.col_idx, Az.val_re[:, 0]
    np.savez_compressed(HERE / "ilu_small.npz", **data)


class HistoryHook:
    """Record every norm2() result inside the method body (not solve()'s
    true-residual norms): SURVEY.md section 4.4 residual-history hook."""

    def __init__(self):
        self.rec = []
        self.active = False
        self._orig = solvers.norm2
        self._disp = dict(solvers._DISPATCH)

    def __enter__(self):
        def norm2(v):
            r = self._orig(v)
            if self.active:
                self.rec.append(r.components)
            return r

        def wrap(fn):
            def inner(*a, **kw):
                self.active = True
                try:
                    return fn(*a, **kw)
                finally:
                    self.active = False
            return inner

        solvers.norm2 = norm2
        for m, fn in self._disp.items():
            solvers._DISPATCH[m] = wrap(fn)
        return self

    def __exit__(self, *exc):
        solvers.norm2 = self._orig
        solvers._DISPATCH.update(self._disp)


def run_ref(A64_re, A64_im, rp, ci, n, b, method, k, eps_rel, eps_abs, max_iter,
            precond="ilu0-mixed", spmv_mode="mixed"):
    prec = PREC[k]
    vre = np.zeros((len(ci), k))
    vre[:, 0] = A64_re
    vim = None
    if A64_im is not None:
        vim = np.zeros((len(ci), k))
        vim[:, 0] = A64_im
    A = sparse.CsrMatrix(n, rp, ci, vre, vim, prec)
    cfg = solvers.SolverConfig(method=method, precision=prec,
                               precond=ilu.PrecondMode(precond), spmv_mode=spmv_mode,
                               eps_rel=eps_rel, eps_abs=eps_abs, max_iter=max_iter)
    with HistoryHook() as hk:
        t0 = time.perf_counter()
        rep = solvers.solve(A, b, cfg)
        dt = time.perf_counter() - t0
    hist = np.array(hk.rec) if hk.rec else np.zeros((0, k))
    out = {
        "iterations": np.array(rep.iterations),
        "converged": np.array(rep.converged),
        "breakdown": np.array(rep.breakdown or ""),
        "final_recursive_relres": np.array(rep.final_recursive_relres),
        "true_relres": np.array(rep.true_relres),
        "hist": hist,
        "seconds": np.array(dt),
    }
    if rep.x is not None:
        out["x_re"] = rep.x.re
        if rep.x.im is not None:
            out["x_im"] = rep.x.im
    return out


def rhs(A64_re, A64_im, rp, ci, n, k, x_true=None, b64=None):
    prec = PREC[k]
    A64 = sparse.CsrMatrix(n, rp, ci, A64_re[:, None],
                           None if A64_im is None else A64_im[:, None], Precision.F64)
    if b64 is not None:
        return sparse.DenseVector.from_float64(b64, prec)
    return sparse.spmv_mixed(A64, sparse.DenseVector.from_float64(x_true, prec))


def gen_solver_small():
    data = {}
    for cx in (False, True):
        tag = "c" if cx else "r"
        rng = np.random.default_rng(31 if not cx else 32)
        A64 = random_dd(rng, 60, 0.12, cx)
        n = A64.n
        xt = rng.uniform(-1, 1, n) + (1j * rng.uniform(-1, 1, n) if cx else 0.0)
        data[f"{tag}_rp"], data[f"{tag}_ci"] = A64.row_ptr, A64.col_idx
        data[f"{tag}_vre"] = A64.val_re[:, 0]
        vim = A64.val_im[:, 0] if cx else None
        if cx:
            data[f"{tag}_vim"] = vim
        data[f"{tag}_xtrue"] = xt
        for k in (2, 3, 4):
            b = rhs(A64.val_re[:, 0], vim, A64.row_ptr, A64.col_idx, n, k, x_true=xt)
            data[f"{tag}{k}_b_re"] = b.re
            if cx:
                data[f"{tag}{k}_b_im"] = b.im
            tol = {2: 1e-25, 3: 1e-40, 4: 1e-55}[k]
            for m in ("bicg", "cgs", "bicgstab", "gpbicg"):
                o = run_ref(A64.val_re[:, 0], vim, A64.row_ptr, A64.col_idx, n, b, m, k,
                            tol, 1e-100, None)
                for key, v in o.items():
                    data[f"{tag}{k}_{m}_{key}"] = v
    np.savez_compressed(HERE / "solver_small.npz", **data)


def gen_solver_none():
    """the unpreconditioned path (precond='none',
    M = I, solvers.py:128-136) in mixed SpMV mode, and spmv_mode='full' with
    ILU(0)-mixed on a binary64 matrix at working precision, on the
    solver_small systems."""
    data = {}
    for cx in (False, True):
        tag = "c" if cx else "r"
        rng = np.random.default_rng(31 if not cx else 32)
        A64 = random_dd(rng, 60, 0.12, cx)
        n = A64.n
        xt = rng.uniform(-1, 1, n) + (1j * rng.uniform(-1, 1, n) if cx else 0.0)
        vim = A64.val_im[:, 0] if cx else None
        for k in (2, 3):
            b = rhs(A64.val_re[:, 0], vim, A64.row_ptr, A64.col_idx, n, k, x_true=xt)
            tol = {2: 1e-25, 3: 1e-40}[k]
            for m in ("bicg", "cgs", "bicgstab", "gpbicg"):
                o = run_ref(A64.val_re[:, 0], vim, A64.row_ptr, A64.col_idx, n, b, m, k,
                            tol, 1e-100, None, precond="none")
                for key, v in o.items():
                    data[f"{tag}{k}_none_{m}_{key}"] = v
            for m in ("bicg", "cgs", "bicgstab", "gpbicg"):
                o = run_ref(A64.val_re[:, 0], vim, A64.row_ptr, A64.col_idx, n, b, m, k,
                            tol, 1e-100, None, spmv_mode="full")
                for key, v in o.items():
                    data[f"{tag}{k}_full_{m}_{key}"] = v
    np.savez_compressed(HERE / "solver_none.npz", **data)


def gen_grid():
    """the reference harness's problem construction
    (bench.build_problem) and its default grid on a small real matrix."""
    from mpkrylov import bench as rbench

    data = {}
    rp, ci, v = problems.convdiff5(8, 10.0)[:3]
    n = len(rp) - 1
    crp, cci, cvr, cvi = problems.helmholtz7(4, 7)[:4]
    nc = len(crp) - 1
    for k in (2, 3):
        vre = np.zeros((len(ci), k))
        vre[:, 0] = v
        A = sparse.CsrMatrix(n, rp, ci, vre, None, PREC[k])
        pr = rbench.build_problem(A, PREC[k], "cd5_8")
        data[f"r{k}_xstar"], data[f"r{k}_b"] = pr.x_star.re, pr.b.re
        vr = np.zeros((len(cci), k))
        vi = np.zeros((len(cci), k))
        vr[:, 0], vi[:, 0] = cvr, cvi
        C = sparse.CsrMatrix(nc, crp, cci, vr, vi, PREC[k])
        pc = rbench.build_problem(C, PREC[k], "helm4")
        data[f"c{k}_xstar_re"], data[f"c{k}_xstar_im"] = pc.x_star.re, pc.x_star.im
        data[f"c{k}_b_re"], data[f"c{k}_b_im"] = pc.b.re, pc.b.im
    vre = np.zeros((len(ci), 2))
    vre[:, 0] = v
    A = sparse.CsrMatrix(n, rp, ci, vre, None, Precision.DD)
    pr = rbench.build_problem(A, Precision.DD, "cd5_8")
    suite = [(A, pr, solvers.SolverConfig(method=m, precision=p, precond=pre, spmv_mode=mode,
                                          eps_rel=1e-20))
             for m, p, pre, mode in rbench.default_grid(precisions=[Precision.DD])]
    rows = rbench.run_benchmark(suite)
    data["grid_iterations"] = np.array([r.iterations for r in rows])
    data["grid_converged"] = np.array([r.converged for r in rows])
    data["grid_keys"] = np.array([f"{r.method}|{r.precond}|{r.spmv_mode}" for r in rows])
    data["grid_true_relres"] = np.array([r.true_relres for r in rows])
    data["grid_err2"] = np.array([r.err2 for r in rows])
    np.savez_compressed(HERE / "grid_small.npz", **data)


def gen_ilu_full():
    """working-precision ILU(0) ('ilu0', ilu.py:279-281)
    factors, applies and solves on the solver_small real system, plus the
    cfg1 (convection-diffusion, k=2) factors and one apply."""
    data = {}
    rng = np.random.default_rng(31)
    A64 = random_dd(rng, 60, 0.12, False)
    n = A64.n
    xt = rng.uniform(-1, 1, n)
    r2 = np.random.default_rng(7)
    for k in (2, 3, 4):
        vre = np.zeros((len(A64.col_idx), k))
        vre[:, 0] = A64.val_re[:, 0]
        A = sparse.CsrMatrix(n, A64.row_ptr, A64.col_idx, vre, None, PREC[k])
        F = ilu.ilu0_factorize(A)
        data[f"k{k}_lu"] = F.val_re
        rv = np.array([rand_mc(r2, k) for _ in range(n)])
        data[f"k{k}_r"] = rv
        data[f"k{k}_z"] = ilu.ilu0_apply(F, sparse.DenseVector(rv.copy(), None, PREC[k])).re
        data[f"k{k}_zadj"] = ilu.ilu0_apply_adjoint(
            F, sparse.DenseVector(rv.copy(), None, PREC[k])).re
        if k in (2, 3):
            b = rhs(A64.val_re[:, 0], None, A64.row_ptr, A64.col_idx, n, k, x_true=xt)
            tol = {2: 1e-25, 3: 1e-40}[k]
            for m in ("bicg", "cgs", "bicgstab", "gpbicg"):
                o = run_ref(A64.val_re[:, 0], None, A64.row_ptr, A64.col_idx, n, b, m, k,
                            tol, 1e-100, None, precond="ilu0")
                for key, v in o.items():
                    data[f"k{k}_{m}_{key}"] = v
    # complex: the solver_small "c" system
    rng = np.random.default_rng(32)
    C64 = random_dd(rng, 60, 0.12, True)
    nc = C64.n
    xtc = rng.uniform(-1, 1, nc) + 1j * rng.uniform(-1, 1, nc)
    for k in (2, 3, 4):
        vre = np.zeros((len(C64.col_idx), k))
        vim = np.zeros((len(C64.col_idx), k))
        vre[:, 0] = C64.val_re[:, 0]
        vim[:, 0] = C64.val_im[:, 0]
        A = sparse.CsrMatrix(nc, C64.row_ptr, C64.col_idx, vre, vim, PREC[k])
        F = ilu.ilu0_factorize(A)
        data[f"c{k}_lu_re"], data[f"c{k}_lu_im"] = F.val_re, F.val_im
        rr = np.array([rand_mc(r2, k) for _ in range(nc)])
        ri = np.array([rand_mc(r2, k) for _ in range(nc)])
        data[f"c{k}_r_re"], data[f"c{k}_r_im"] = rr, ri
        z = ilu.ilu0_apply(F, sparse.DenseVector(rr.copy(), ri.copy(), PREC[k]))
        data[f"c{k}_z_re"], data[f"c{k}_z_im"] = z.re, z.im
        za = ilu.ilu0_apply_adjoint(F, sparse.DenseVector(rr.copy(), ri.copy(), PREC[k]))
        data[f"c{k}_zadj_re"], data[f"c{k}_zadj_im"] = za.re, za.im
        if k in (2, 3):
            b = rhs(C64.val_re[:, 0], C64.val_im[:, 0], C64.row_ptr, C64.col_idx, nc, k,
                    x_true=xtc)
            tol = {2: 1e-25, 3: 1e-40}[k]
            for m in ("bicg", "cgs", "bicgstab", "gpbicg"):
                o = run_ref(C64.val_re[:, 0], C64.val_im[:, 0], C64.row_ptr, C64.col_idx, nc, b,
                            m, k, tol, 1e-100, None, precond="ilu0")
                for key, v in o.items():
                    data[f"c{k}_{m}_{key}"] = v
    p = problems.cfg1()
    vre = np.zeros((p.nnz, 2))
    vre[:, 0] = p.val_re
    A = sparse.CsrMatrix(p.n, p.row_ptr, p.col_idx, vre, None, Precision.DD)
    F = ilu.ilu0_factorize(A)
    data["cfg1_lu"] = F.val_re
    rv = np.array([rand_mc(r2, 2) for _ in range(p.n)])
    data["cfg1_r"] = rv
    data["cfg1_z"] = ilu.ilu0_apply(F, sparse.DenseVector(rv.copy(), None, Precision.DD)).re
    np.savez_compressed(HERE / "ilu_full.npz", **data)


def gen_mc_fused():
    """_mcfast fused sweep primitives (rmulsubK / rmulK) of the working-
    precision ILU(0) on seeded MC operands, incl. cancellation a ~ b*c."""
    from mpkrylov import _mcfast

    data = {}
    rng = np.random.default_rng(91)
    for k in (2, 3, 4):
        A, B, C, MS, MU = [], [], [], [], []
        for t in range(400):
            a, b, c = rand_mc(rng, k, 10.0 ** rng.integers(-8, 9)), rand_mc(rng, k), rand_mc(rng, k)
            if t % 4 == 1:  # near-total cancellation
                a = _mcfast._RMUL[k](b, c)
                a = _mccore.renorm_terms(list(a) + [rng.standard_normal() * 1e-40], k)
            if t % 8 == 3:
                a = (0.0,) * k
            A.append(a)
            B.append(b)
            C.append(c)
            MS.append(_mcfast._RMULSUB[k](a, b, c))
            MU.append(_mcfast._RMUL[k](a, b))
        data[f"k{k}_a"], data[f"k{k}_b"], data[f"k{k}_c"] = np.array(A), np.array(B), np.array(C)
        data[f"k{k}_mulsub"], data[f"k{k}_mul"] = np.array(MS), np.array(MU)
    np.savez_compressed(HERE / "mc_fused.npz", **data)


def mm_texts():
    """Synthetic Matrix Market files for the f3 fixtures: every field /
    symmetry, duplicated entries (exact MC sums), comments, blank lines."""
    rng = np.random.default_rng(77)
    out = {}
    for field in ("real", "integer", "complex", "pattern"):
        for sym in ("general", "symmetric", "hermitian", "skew-symmetric"):
            if sym == "hermitian" and field != "complex":
                continue
            n = 7
            ents = []
            for _ in range(18):
                i, j = sorted(rng.integers(1, n + 1, 2), reverse=True)
                if sym == "skew-symmetric" and i == j:
                    continue
                if sym == "general" and rng.random() < 0.5:
                    i, j = j, i
                if field == "pattern":
                    ents.append(f"{i} {j}")
                elif field == "integer":
                    ents.append(f"{i} {j} {int(rng.integers(-9, 10))}")
                elif field == "complex":
                    ents.append(f"{i} {j} {rng.standard_normal():.17g} {rng.standard_normal():.17g}")
                else:
                    # duplicates with widely different magnitudes: MC sums matter
                    v = rng.standard_normal() * 10.0 ** int(rng.integers(-20, 20))
                    ents.append(f"{i} {j} {v:.17g}")
            for d in range(1, n + 1):
                if sym != "skew-symmetric":
                    if field == "pattern":
                        ents.append(f"{d} {d}")
                    elif field == "complex":
                        ents.append(f"{d} {d} {float(n + d)} 0.0")
                    else:
                        ents.append(f"{d} {d} {n + d}")
            text = (f"%%MatrixMarket matrix coordinate {field} {sym}\n% generated\n\n"
                    f"{n} {n} {len(ents)}\n" + "\n".join(ents) + "\n")
            out[f"{field}_{sym}"] = text
    return out


def gen_mm():
    from mpkrylov import coo_to_csr, parse_matrix_market

    data = {}
    for tag, text in mm_texts().items():
        data[f"{tag}_text"] = np.array(text)
        coo = parse_matrix_market(text)
        data[f"{tag}_coo_row"], data[f"{tag}_coo_col"] = coo.row, coo.col
        data[f"{tag}_coo_re"] = coo.val_re
        for k in (1, 2, 3, 4):
            A = coo_to_csr(coo, PREC[k] if k > 1 else Precision.F64)
            data[f"{tag}_{k}_rp"], data[f"{tag}_{k}_ci"] = A.row_ptr, A.col_idx
            data[f"{tag}_{k}_re"] = A.val_re
            if A.val_im is not None:
                data[f"{tag}_{k}_im"] = A.val_im
    np.savez_compressed(HERE / "mm_small.npz", **data)


def gen_solver_cfg(which):
    data = {}
    if "cfg1" in which:
        p = problems.cfg1()
        data["cfg1_checksum"] = np.array(p.checksum())
        b = rhs(p.val_re, None, p.row_ptr, p.col_idx, p.n, 2, x_true=p.x_true)
        data["cfg1_b_re"] = b.re
        o = run_ref(p.val_re, None, p.row_ptr, p.col_idx, p.n, b, "bicgstab", 2,
                    p.eps_rel, p.eps_abs, p.max_iter)
        for key, v in o.items():
            data[f"cfg1_bicgstab_dd_{key}"] = v
        print("cfg1", o["iterations"], o["seconds"], flush=True)
    if "cfg2" in which:
        p = problems.cfg2()
        data["cfg2_checksum"] = np.array(p.checksum())
        for lab in ("td", "qd"):
            k = LABEL[lab]
            b = rhs(p.val_re, None, p.row_ptr, p.col_idx, p.n, k, x_true=p.x_true)
            data[f"cfg2_{lab}_b_head"] = b.re[:64]
            for m in p.methods:
                o = run_ref(p.val_re, None, p.row_ptr, p.col_idx, p.n, b, m, k,
                            p.eps_rel, p.eps_abs, p.max_iter)
                o.pop("x_re", None)
                for key, v in o.items():
                    data[f"cfg2_{m}_{lab}_{key}"] = v
                print("cfg2", m, lab, o["iterations"], o["seconds"], flush=True)
    if "cfg3" in which:
        p = problems.cfg3()
        data["cfg3_checksum"] = np.array(p.checksum())
        b = rhs(p.val_re, p.val_im, p.row_ptr, p.col_idx, p.n, 2, b64=p.b64)
        for m in p.methods:
            o = run_ref(p.val_re, p.val_im, p.row_ptr, p.col_idx, p.n, b, m, 2,
                        p.eps_rel, p.eps_abs, 20)
            o.pop("x_re", None)
            o.pop("x_im", None)
            for key, v in o.items():
                data[f"cfg3_{m}_dd_{key}"] = v
            print("cfg3", m, o["iterations"], o["seconds"], flush=True)
    if "cfg5" in which:
        p = problems.cfg5(0)
        data["cfg5_0_checksum"] = np.array(p.checksum())
        b = rhs(p.val_re, None, p.row_ptr, p.col_idx, p.n, 4, x_true=p.x_true)
        for m in p.methods:
            o = run_ref(p.val_re, None, p.row_ptr, p.col_idx, p.n, b, m, 4,
                        p.eps_rel, p.eps_abs, p.max_iter)
            o.pop("x_re", None)
            for key, v in o.items():
                data[f"cfg5_0_{m}_qd_{key}"] = v
            print("cfg5", m, o["iterations"], o["seconds"], flush=True)
    name = "solver_" + "_".join(which) + ".npz"
    np.savez_compressed(HERE / name, **data)


if __name__ == "__main__":
    what = sys.argv[1:] or ["mc", "sparse", "ilu", "small", "cfg"]
    t0 = time.time()
    if "mc" in what:
        gen_mc_ops()
        print("mc_ops done", time.time() - t0, flush=True)
    if "sparse" in what:
        gen_sparse()
        print("sparse done", time.time() - t0, flush=True)
    if "ilu" in what:
        gen_ilu()
        print("ilu done", time.time() - t0, flush=True)
    if "small" in what:
        gen_solver_small()
        print("solver_small done", time.time() - t0, flush=True)
    if "grid" in what:
        gen_grid()
        print("grid done", time.time() - t0, flush=True)
    if "ilufull" in what:
        gen_ilu_full()
        print("ilufull done", time.time() - t0, flush=True)
    if "fused" in what:
        gen_mc_fused()
        print("fused done", time.time() - t0, flush=True)
    if "mm" in what:
        gen_mm()
        print("mm done", time.time() - t0, flush=True)
    if "none" in what:
        gen_solver_none()
        print("solver_none done", time.time() - t0, flush=True)
    for c in ("cfg1", "cfg2", "cfg3", "cfg5"):
        if "cfg" in what or c in what:
            gen_solver_cfg([c])
            print(c, "done", time.time() - t0, flush=True)
