"""Full-size parity fixtures from the pinned C ORACLE (run here only).

    python tests/golden/make_oracle_full.py [cfg3] [cfg5] [cfg4]

The unmodified Python reference needs hours for these solves (cfg3: ~2.6 s
per iteration and ~1400 iterations; cfg5: 128 QD solves of ~30 s; cfg4:
~36 s per iteration), so these fixtures come from oracle/mpk_oracle.c, the
C restatement of the reference that tests/test_oracle_golden.py pins bit
for bit to reference-generated vectors (every MC op, SpMV, ILU(0), and the
full solves of cfg1, cfg2, cfg3 (20 it), cfg5 system 0), and for cfg4
to tests/golden/cfg4_ref.npz (reference-generated factors, apply and
20-iteration history; tests/test_oracle_golden.py::test_oracle_cfg4_*).

Written: tests/golden/full_cfg3.npz, full_cfg5.npz, full_cfg4.npz with, per
solve, iterations / converged / breakdown / true relres / the first 41
norm2-history entries (= the first 20 iterations for every method), and
for cfg4 the whole 200-iteration history.
"""

from __future__ import annotations

import pathlib
import sys
import time

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_2504_14498_b200 import problems  # noqa: E402

NH = 41


def _rhs(p, k):
    n = p.n
    cx = p.val_im is not None
    if p.b64 is not None:
        b_re = np.zeros((n, k))
        b_re[:, 0] = np.real(p.b64)
        b_im = None
        if cx:
            b_im = np.zeros((n, k))
            b_im[:, 0] = np.imag(p.b64)
        return b_re, b_im
    x = np.zeros((n, k))
    x[:, 0] = np.real(p.x_true)
    xi = None
    if cx:
        xi = np.zeros((n, k))
        xi[:, 0] = np.imag(p.x_true)
    return oracle.spmv_mixed(n, p.row_ptr, p.col_idx, p.val_re, p.val_im, x, xi)


def _solve(p, m, k, max_iter=None, nh=NH):
    b_re, b_im = _rhs(p, k)
    mi = max_iter if max_iter is not None else (p.max_iter or 3 * p.n)
    t0 = time.perf_counter()
    rep, x_re, x_im, hist = oracle.solve(p.n, p.row_ptr, p.col_idx, p.val_re, p.val_im, m,
                                         k, b_re, b_im, eps_rel=p.eps_rel,
                                         eps_abs=p.eps_abs, max_iter=mi)
    dt = time.perf_counter() - t0
    h = np.zeros((nh, k))
    h[: min(nh, len(hist))] = hist[:nh]
    return {"iterations": np.array(rep.iterations), "converged": np.array(rep.converged),
            "breakdown": np.array(oracle.BREAKDOWN[rep.breakdown] or ""),
            "true_relres": np.array(rep.true_relres),
            "final_recursive_relres": np.array(rep.final_recursive_relres),
            "hist_len": np.array(len(hist)), "hist": h, "seconds": np.array(dt)}


def gen_cfg3():
    p = problems.cfg3()
    data = {"checksum": np.array(p.checksum())}
    for m in p.methods:
        o = _solve(p, m, 2)
        for key, v in o.items():
            data[f"{m}_dd_{key}"] = v
        print("cfg3", m, int(o["iterations"]), bool(o["converged"]), float(o["true_relres"]),
              f"{float(o['seconds']):.1f}s", flush=True)
    np.savez_compressed(HERE / "full_cfg3.npz", **data)


def gen_cfg5(nsys=64):
    data = {}
    for s in range(nsys):
        p = problems.cfg5(s)
        data[f"s{s}_checksum"] = np.array(p.checksum())
        for m in p.methods:
            o = _solve(p, m, 4)
            for key, v in o.items():
                data[f"s{s}_{m}_qd_{key}"] = v
            print("cfg5", s, m, int(o["iterations"]), bool(o["converged"]),
                  f"{float(o['seconds']):.1f}s", flush=True)
    np.savez_compressed(HERE / "full_cfg5.npz", **data)


def gen_cfg4():
    p = problems.cfg4()
    o = _solve(p, "bicgstab", 2, max_iter=200, nh=2 * 200 + 2)
    data = {"checksum": np.array(p.checksum())}
    for key, v in o.items():
        data[f"bicgstab_dd_{key}"] = v
    print("cfg4", int(o["iterations"]), f"{float(o['seconds']):.1f}s", flush=True)
    np.savez_compressed(HERE / "full_cfg4.npz", **data)


if __name__ == "__main__":
    what = sys.argv[1:] or ["cfg3", "cfg5", "cfg4"]
    oracle.set_threads(int(__import__("os").environ.get("ORC_THREADS", "6")))
    if "cfg3" in what:
        gen_cfg3()
    if "cfg5" in what:
        gen_cfg5()
    if "cfg4" in what:
        gen_cfg4()
