import sys, time, pathlib
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2504_14498_b200 as pkg
from paper_2504_14498_b200 import problems
p = problems.cfg2()
for k, P in ((3, pkg.Precision.TD), (4, pkg.Precision.QD)):
    A = pkg.CsrMatrix.from_binary64(p.n, p.row_ptr, p.col_idx, p.val_re, None, P)
    b = pkg.spmv_mixed(A.demoted(), pkg.DenseVector.from_float64(p.x_true, P))
    for m in ("bicg", "bicgstab"):
        for pre in (pkg.PrecondMode.ILU0_MIXED, pkg.PrecondMode.ILU0_FULL):
            cfg = pkg.SolverConfig(method=m, precision=P, precond=pre, spmv_mode="mixed", eps_rel=p.eps_rel, max_iter=p.max_iter)
            pkg.solve(A, b, cfg)
            r = pkg.solve(A, b, cfg)
            print(k, m, pre.value, r.iterations, r.converged, r.breakdown, "%.2e" % r.final_recursive_relres, "%.2e" % r.true_relres, "factor %.2f ms solve %.2f ms per-it %.3f ms" % (r.factor_seconds*1e3, r.solve_seconds*1e3, r.solve_seconds*1e3/max(r.iterations,1)))
