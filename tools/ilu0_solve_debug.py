import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2504_14498_b200 as pkg
from paper_2504_14498_b200 import problems
p = problems.cfg2()
k, P = 3, pkg.Precision.TD
A = pkg.CsrMatrix.from_binary64(p.n, p.row_ptr, p.col_idx, p.val_re, None, P)
b = pkg.spmv_mixed(A.demoted(), pkg.DenseVector.from_float64(p.x_true, P))
for m in sys.argv[1:] or ["bicg", "bicgstab", "cgs", "gpbicg"]:
    cfg = pkg.SolverConfig(method=m, precision=P, precond=pkg.PrecondMode.ILU0_FULL, spmv_mode="mixed",
                           eps_rel=p.eps_rel, max_iter=p.max_iter)
    out = []
    for t in range(4):
        r = pkg.solve(A, b, cfg)
        out.append((r.iterations, r.converged, r.breakdown, r.history[:3]))
    print(m, [(o[0], o[1], o[2]) for o in out])
    print("  first hist", out[0][3])
