import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2504_14498_b200 as pkg
from paper_2504_14498_b200 import problems, _lib
p = problems.cfg2()
k, P = 2, pkg.Precision.DD
A = pkg.CsrMatrix.from_binary64(p.n, p.row_ptr, p.col_idx, p.val_re, None, P)
b = pkg.spmv_mixed(A.demoted(), pkg.DenseVector.from_float64(p.x_true, P))
cfg = pkg.SolverConfig(method="bicg", precision=P, precond=pkg.PrecondMode.ILU0_FULL, spmv_mode="mixed",
                       eps_rel=1e-20, max_iter=100)
for t in range(3):
    r = pkg.solve(A, b, cfg)
    print(t, r.iterations, r.converged, r.breakdown, [h[0] for h in r.history[:4]])
# standalone applies after solves
F = pkg.ilu0_factorize(A)
rng = np.random.default_rng(1)
rv = pkg.DenseVector(rng.standard_normal((p.n, k)) * np.array([1, 1e-17]), None, P)
for t in range(3):
    z = pkg.ilu0_apply_adjoint(F, rv).re
    print("adj apply finite", np.isfinite(z).all())
