"""Residual-history deviation from the reference goldens, per solver cell,
as a fraction of the north-star bound (first 20 iterations; all iterations).

    python tools/hist_margin.py
"""
import fractions
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_2504_14498_b200 as pkg  # noqa: E402
from paper_2504_14498_b200 import problems  # noqa: E402
from conftest import golden  # noqa: E402

TOL = {2: 1e-25, 3: 1e-40, 4: 1e-55}
PREC = {2: "DD", 3: "TD", 4: "QD"}


def dev(got, ref, m=None):
    got, ref = np.asarray(got), np.asarray(ref)
    n = min(len(got), len(ref)) if m is None else min(len(got), len(ref), m)
    r0 = fractions.Fraction(ref[0].sum()) if ref.shape[1] < 4 else sum(
        fractions.Fraction(c) for c in ref[0])
    out = 0.0
    for a, b in zip(got[:n], ref[:n]):
        d = abs(sum(fractions.Fraction(c) for c in a) - sum(fractions.Fraction(c) for c in b))
        out = max(out, float(d / r0))
    return out


def cell(p, method, k, g, pre, max_iter=None):
    P = getattr(pkg.Precision, PREC[k])
    A = pkg.CsrMatrix.from_binary64(p.n, p.row_ptr, p.col_idx, p.val_re, p.val_im, P)
    if p.b64 is not None:
        b = pkg.DenseVector.from_float64(p.b64, P)
    else:
        b = pkg.spmv_mixed(A.demoted(), pkg.DenseVector.from_float64(p.x_true, P))
    cfg = pkg.SolverConfig(method=method, precision=P, precond=pkg.PrecondMode.ILU0_MIXED,
                           spmv_mode="mixed", eps_rel=p.eps_rel,
                           max_iter=max_iter or p.max_iter)
    rep = pkg.solve(A, b, cfg)
    ref = g[f"{pre}_hist"]
    d20 = dev(rep.history, ref, 41)
    dall = dev(rep.history, ref)
    it_ref = int(g[f"{pre}_iterations"])
    print(f"{pre:24s} it {rep.iterations:4d}/{it_ref:4d}  dev20 {d20:9.2e} ({d20 / TOL[k]:8.1e} of tol)"
          f"  devall {dall:9.2e} ({dall / TOL[k]:8.1e})", flush=True)


def main():
    g = golden("solver_cfg1.npz")
    cell(problems.cfg1(), "bicgstab", 2, g, "cfg1_bicgstab_dd")
    g = golden("solver_cfg2.npz")
    p = problems.cfg2()
    for lab, k in (("td", 3), ("qd", 4)):
        for m in ("bicg", "cgs", "bicgstab", "gpbicg"):
            cell(p, m, k, g, f"cfg2_{m}_{lab}")
    g = golden("solver_cfg5.npz")
    for m in ("cgs", "bicgstab"):
        cell(problems.cfg5(0), m, 4, g, f"cfg5_0_{m}_qd")
    g = golden("solver_cfg3.npz")
    for m in ("bicgstab", "gpbicg"):
        cell(problems.cfg3(), m, 2, g, f"cfg3_{m}_dd", max_iter=20)


if __name__ == "__main__":
    main()
