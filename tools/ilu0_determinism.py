"""Working-precision ILU(0) applies on cfg2: repeated plain / adjoint applies
must be bitwise identical and finite (race detector for the K-component
sweeps)."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2504_14498_b200 as pkg
from paper_2504_14498_b200 import problems
p = problems.cfg2()
for k, P in ((3, pkg.Precision.TD), (4, pkg.Precision.QD)):
    A = pkg.CsrMatrix.from_binary64(p.n, p.row_ptr, p.col_idx, p.val_re, None, P)
    F = pkg.ilu0_factorize(A)
    F2 = pkg.ilu0_factorize(A)
    print(k, "factors finite", np.isfinite(F.val_re).all(), "repeat-equal", np.array_equal(F.val_re, F2.val_re))
    rng = np.random.default_rng(3)
    r = pkg.DenseVector(rng.standard_normal((p.n, k)) * np.array([1, 1e-17, 1e-34, 1e-51][:k]), None, P)
    for name, fn in (("plain", pkg.ilu0_apply), ("adjoint", pkg.ilu0_apply_adjoint)):
        z0 = fn(F, r).re
        bad = 0
        for t in range(20):
            z = fn(F, r).re
            bad += int(not np.array_equal(z, z0))
        print(k, name, "finite", np.isfinite(z0).all(), "max|z|", np.abs(z0[:, 0]).max(), "mismatches", bad)
