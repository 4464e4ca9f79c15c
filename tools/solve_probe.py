"""One short solve of a BASELINE config through the public API (ncu target: run it with
MPK_NO_COND_GRAPH=1 so the iteration's kernels are plain graph nodes ncu can profile).

usage: python tools/solve_probe.py cfg4 [iterations] [method] [precision label]
"""
import pathlib
import sys
import time

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_2504_14498_b200 as mpk  # noqa: E402
from paper_2504_14498_b200 import problems  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 10
method = sys.argv[3] if len(sys.argv) > 3 else "bicgstab"
P = mpk.Precision.from_label(sys.argv[4]) if len(sys.argv) > 4 else mpk.Precision.DD
p = problems.CONFIGS[name](0) if name == "cfg5" else problems.CONFIGS[name]()
A = mpk.CsrMatrix.from_binary64(p.n, p.row_ptr, p.col_idx, p.val_re, p.val_im, P)
if p.x_true is not None:
    b = mpk.spmv_mixed(A.demoted(), mpk.DenseVector.from_float64(p.x_true, P))
else:
    b = mpk.DenseVector.from_float64(p.b64, P)
cfg = mpk.SolverConfig(method=method, precision=P, precond=mpk.PrecondMode.ILU0_MIXED,
                       spmv_mode="mixed", eps_rel=1e-300, max_iter=its)
t0 = time.perf_counter()
rep = mpk.solve(A, b, cfg)
print(name, method, P.label, "iterations", rep.iterations, "converged", rep.converged,
      "breakdown", rep.breakdown, "relres", rep.final_recursive_relres, "wall s",
      round(time.perf_counter() - t0, 3), "solve_seconds", rep.solve_seconds)
