"""Golden vectors for MC-valued matrices, from the REFERENCE (run here only).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_mcmat.py

An MC-valued matrix has non-zero tail components (e.g. Matrix Market input
with duplicate entries summed in working precision, sparse.py:308-319), so
its SpMV multiplies MC x MC (sparse.py:414-451, _kernels.py:224-240,
266-278, 300-323, 356-376) and only spmv_mode='full' accepts it
(solvers.py:120-123).  Records, on seeded inputs: spmv / spmv_adjoint,
scale / vec_sub / vec_add, the working-precision ILU(0) factors of the
MC-valued matrix, and full solver runs (spmv_mode='full' with ILU(0)-mixed
on the demoted matrix, with no preconditioner and with the
working-precision ILU(0)) with their residual histories.  Also one Matrix
Market text with duplicate entries whose CSR values are MC-valued, and its
DD BiCGSTAB run.  Writes mcmat.npz next to this script.
"""

from __future__ import annotations

import sys
import time

import numpy as np

import make_golden as mg
from make_golden import HERE, PREC, HistoryHook, ilu, mc_vec, mpkrylov, rand_mc, random_dd, solvers, sparse
from mpkrylov import _mccore


def mc_values(rng, heads, k):
    """k-component values whose head is (close to) the given binary64 value
    and whose tails carry content in every limb."""
    out = np.zeros((len(heads), k))
    for p, h in enumerate(heads):
        terms = [float(h)] + [float(h) * rng.uniform(-1.0, 1.0) * 2.0 ** (-53 * i)
                              for i in range(1, k)]
        out[p] = _mccore.renormalize(terms, k)
    return out


def run_ref_mc(A, b, method, k, eps_rel, precond, max_iter=None):
    cfg = solvers.SolverConfig(method=method, precision=PREC[k],
                               precond=ilu.PrecondMode(precond), spmv_mode="full",
                               eps_rel=eps_rel, eps_abs=1e-100, max_iter=max_iter)
    with HistoryHook() as hk:
        rep = solvers.solve(A, b, cfg)
    out = {
        "iterations": np.array(rep.iterations),
        "converged": np.array(rep.converged),
        "breakdown": np.array(rep.breakdown or ""),
        "true_relres": np.array(rep.true_relres),
        "hist": np.array(hk.rec) if hk.rec else np.zeros((0, k)),
    }
    if rep.x is not None:
        out["x_re"] = rep.x.re
        if rep.x.im is not None:
            out["x_im"] = rep.x.im
    return out


MM_DUP = """%%MatrixMarket matrix coordinate real general
% duplicate entries: their working-precision sums are not binary64 values
4 4 11
1 1 4.0
1 1 1e-20
1 2 -1.0
2 1 -1.0
2 2 4.0
2 2 3e-19
2 3 -1.0
3 2 -1.0
3 3 4.0
3 4 0.1
4 4 5.0
"""


def main():
    data = {}
    t0 = time.time()
    for cx in (False, True):
        tag = "c" if cx else "r"
        rng = np.random.default_rng(41 if not cx else 42)
        A64 = random_dd(rng, 60, 0.12, cx)
        n = A64.n
        data[f"{tag}_rp"], data[f"{tag}_ci"] = A64.row_ptr, A64.col_idx
        xt = rng.uniform(-1, 1, n) + (1j * rng.uniform(-1, 1, n) if cx else 0.0)
        for k in (2, 3, 4):
            P = PREC[k]
            vre = mc_values(rng, A64.val_re[:, 0], k)
            vim = mc_values(rng, A64.val_im[:, 0], k) if cx else None
            A = sparse.CsrMatrix(n, A64.row_ptr, A64.col_idx, vre, vim, P)
            data[f"{tag}{k}_vre"] = vre
            if cx:
                data[f"{tag}{k}_vim"] = vim
            x, y = mc_vec(rng, n, k, cx), mc_vec(rng, n, k, cx)
            s, sa = sparse.spmv(A, x), sparse.spmv_adjoint(A, x)
            if cx:
                al = mpkrylov.MCComplex(mpkrylov.MCFloat(rand_mc(rng, k)),
                                        mpkrylov.MCFloat(rand_mc(rng, k)))
                data[f"{tag}{k}_alpha_re"] = np.array(al.re.components)
                data[f"{tag}{k}_alpha_im"] = np.array(al.im.components)
            else:
                al = mpkrylov.MCFloat(rand_mc(rng, k))
                data[f"{tag}{k}_alpha_re"] = np.array(al.components)
            sc, vs, va = sparse.scale(al, x), sparse.vec_sub(x, y), sparse.vec_add(x, y)
            for name, v in (("x", x), ("y", y), ("spmv", s), ("adj", sa), ("scale", sc),
                            ("sub", vs), ("add", va)):
                data[f"{tag}{k}_{name}_re"] = v.re
                if cx:
                    data[f"{tag}{k}_{name}_im"] = v.im
            F = ilu.ilu0_factorize(A)
            data[f"{tag}{k}_lu_re"] = F.val_re
            if cx:
                data[f"{tag}{k}_lu_im"] = F.val_im
            if k == 4:
                continue
            b = sparse.spmv(A, sparse.DenseVector.from_float64(xt, P))
            data[f"{tag}{k}_b_re"] = b.re
            if cx:
                data[f"{tag}{k}_b_im"] = b.im
            tol = {2: 1e-25, 3: 1e-40}[k]
            cells = [(m, "ilu0-mixed") for m in ("bicg", "cgs", "bicgstab", "gpbicg")]
            cells += [("bicgstab", "none"), ("bicg", "none"), ("bicgstab", "ilu0"),
                      ("gpbicg", "ilu0")]
            for m, pre in cells:
                o = run_ref_mc(A, b, m, k, tol, pre)
                for key, v in o.items():
                    data[f"{tag}{k}_{pre}_{m}_{key}"] = v
            print(tag, k, "done", round(time.time() - t0, 1), flush=True)
    # Matrix Market input with duplicate entries -> MC-valued CSR -> full solve
    coo = sparse.parse_matrix_market(MM_DUP)
    A = sparse.coo_to_csr(coo, PREC[2])
    assert np.any(A.val_re[:, 1:]), "duplicates must leave non-zero tails"
    data["mm_text"] = np.array(MM_DUP)
    data["mm_rp"], data["mm_ci"], data["mm_vre"] = A.row_ptr, A.col_idx, A.val_re
    b = sparse.spmv(A, sparse.DenseVector.from_float64(np.ones(A.n), PREC[2]))
    data["mm_b_re"] = b.re
    o = run_ref_mc(A, b, "bicgstab", 2, 1e-25, "ilu0-mixed")
    for key, v in o.items():
        data[f"mm_bicgstab_{key}"] = v
    np.savez_compressed(HERE / "mcmat.npz", **data)
    print("mcmat done", round(time.time() - t0, 1))


if __name__ == "__main__":
    sys.exit(main())
