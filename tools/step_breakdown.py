"""Per-cell breakdown of one bench step: every cell of a config solved
alone (serial) and all together (mpk_run_jobs), device-resident.

    python tools/step_breakdown.py [cfg2] [--reps 3]
"""
import argparse
import ctypes
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2504_14498_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="cfg2")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    L = _lib.lib()

    def ctx():
        h = ctypes.c_void_p()
        _lib.check(L.mpk_ctx_create(ctypes.c_int(0), ctypes.byref(h)))
        return h

    cells = [bench.Cell(L, _lib, p, m, k, ctx()) for (p, m, k) in bench.cells_for(a.config, 0, 1)]
    J = (_lib.MpkJob * len(cells))()
    for j, c in enumerate(cells):
        J[j].m = c.m; J[j].method = _lib.METHOD_CODE[c.method]; J[j].k = c.k
        J[j].eps_rel = c.p.eps_rel; J[j].eps_abs = c.p.eps_abs; J[j].max_iter = c.max_iter
        J[j].b_re = c.d_b.data_ptr(); J[j].x_re = c.d_x.data_ptr()
        J[j].hist = c.d_h.data_ptr(); J[j].hist_cap = c.hist_cap

    def show(tag):
        for j, c in enumerate(cells):
            r = J[j].rep
            print(f"  {tag} {c.method:9s} k={c.k}: it={r.iterations:4d} factor={r.factor_ms:6.3f} "
                  f"loop={r.solve_ms:7.3f} total={r.total_ms:7.3f} ms  per-it={r.solve_ms / max(r.iterations, 1):.3f}")

    _lib.check(L.mpk_run_jobs(J, len(cells), 1))
    for _ in range(a.reps):
        for j in range(len(cells)):
            _lib.check(L.mpk_run_jobs(ctypes.byref(J[j]), 1, 1))
    show("serial")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.reps):
        _lib.check(L.mpk_run_jobs(J, len(cells), 1))
    torch.cuda.synchronize()
    print(f"concurrent step wall {1e3 * (time.perf_counter() - t0) / a.reps:.2f} ms")
    show("conc")


if __name__ == "__main__":
    main()
