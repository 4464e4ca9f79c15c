"""Time the working-precision ILU(0) path on a bench config: a short
BiCGSTAB solve with precond='ilu0' (factorization + a few iterations),
reported as ms per iteration (tools/, not part of the product)."""
import sys
import time

import numpy as np

import paper_2504_14498_b200 as pkg
from paper_2504_14498_b200 import problems

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 6
p = getattr(problems, cfg_name)()
P = pkg.Precision.DD
A = pkg.CsrMatrix.from_binary64(p.n, p.row_ptr, p.col_idx, p.val_re, p.val_im, P)
b = pkg.DenseVector.from_float64(p.b64, P) if p.b64 is not None else \
    pkg.spmv_mixed(A.demoted(), pkg.DenseVector.from_float64(p.x_true, P))
for it in (1, 1, iters):
    cfg = pkg.SolverConfig(method="bicgstab", precision=P, precond=pkg.PrecondMode.ILU0_FULL,
                           eps_rel=1e-300, eps_abs=1e-300, max_iter=it)
    t0 = time.perf_counter()
    rep = pkg.solve(A, b, cfg)
    t = time.perf_counter() - t0
    print(f"{cfg_name} max_iter={it}: {rep.iterations} it, {t * 1e3:.1f} ms total", flush=True)
    if it == 1:
        t1 = t
print(f"{cfg_name}: {(t - t1) * 1e3 / (iters - 1):.1f} ms per extra iteration")
