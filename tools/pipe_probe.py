"""Span of the shuffle-wavefront sweep phases inside a solve, with and without the
sweep-pipelined SpMV running beside the backward phase (per-group globaltimer stamps of
the last sweep launched; mpk_swf_debug).   python tools/pipe_probe.py [cfg4] [iterations]"""
import ctypes
import os
import pathlib
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import paper_2504_14498_b200 as mpk  # noqa: E402
from paper_2504_14498_b200 import _lib, problems  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 6
p = problems.CONFIGS[name]()
P = mpk.Precision.DD
L = _lib.lib()
for pipe in ("0", "1"):
    os.environ["MPK_PIPE"] = pipe
    A = mpk.CsrMatrix.from_binary64(p.n, p.row_ptr, p.col_idx, p.val_re, None, P)
    b = mpk.spmv_mixed(A.demoted(), mpk.DenseVector.from_float64(p.x_true if p.x_true is not None
                                                                else np.ones(p.n), P))
    cfg = mpk.SolverConfig(method="bicgstab", precision=P, precond=mpk.PrecondMode.ILU0_MIXED,
                           spmv_mode="mixed", eps_rel=1e-300, eps_abs=1e-300, max_iter=its)
    mpk.solve(A, b, cfg)  # plan + graph
    L.mpk_swf_debug(None, ctypes.c_int(1))
    rep = mpk.solve(A, b, cfg)
    buf = (ctypes.c_longlong * (4 * 4096))()
    L.mpk_swf_debug(buf, ctypes.c_int(0))
    a = np.array(buf[:], dtype=np.int64).reshape(2, 4096, 2)
    out = []
    for ph, nm in ((0, "fwd"), (1, "bwd")):
        st, en = a[ph, :, 0], a[ph, :, 1]
        ng = int(np.count_nonzero(st))
        out.append(f"{nm} span {(en[:ng].max() - st[:ng].min()) / 1e3:8.1f} us ({ng} groups)")
    gap = (a[1, :, 0][a[1, :, 0] > 0].min() - a[0, :, 1].max()) / 1e3
    print(f"MPK_PIPE={pipe}: {rep.iterations} it, solve {rep.solve_seconds * 1e3:.2f} ms "
          f"({rep.solve_seconds * 1e3 / max(rep.iterations, 1):.3f} ms/it incl. setup); "
          + "; ".join(out) + f"; fwd end -> bwd start {gap:.1f} us")
    del A
