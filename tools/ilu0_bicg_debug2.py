import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2504_14498_b200 as pkg
from paper_2504_14498_b200 import problems
P = pkg.Precision.TD
for n in (300, 2000, 20000):
    rp, ci, v, xt = problems.random_nonsym(n, 12, 2)
    for fresh in (False, True):
        A = pkg.CsrMatrix.from_binary64(n, rp, ci, v, None, P)
        b = pkg.spmv_mixed(A.demoted(), pkg.DenseVector.from_float64(xt, P))
        cfg = pkg.SolverConfig(method="bicg", precision=P, precond=pkg.PrecondMode.ILU0_FULL,
                               spmv_mode="mixed", eps_rel=1e-30, max_iter=300)
        res = []
        for t in range(3):
            if fresh and t:
                A = pkg.CsrMatrix.from_binary64(n, rp, ci, v, None, P)
            r = pkg.solve(A, b, cfg)
            res.append((r.iterations, r.converged, r.breakdown))
        print(n, "fresh" if fresh else "same", res, flush=True)
