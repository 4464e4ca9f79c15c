"""Benchmark grid on the device: the reference harness's
problem construction bit for bit and its default grid (4 methods x DD x
{plain, ILU(0), mixed SpMV, mixed SpMV + ILU(0)_d}) with the reference's
iteration counts (twin-mode reductions), against tests/golden/grid_small.npz."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import bits_equal, golden

pytestmark = pytest.mark.gpu


def _mats(pkg, k):
    from paper_2504_14498_b200 import problems

    P = {2: pkg.Precision.DD, 3: pkg.Precision.TD}[k]
    rp, ci, v = problems.convdiff5(8, 10.0)[:3]
    A = pkg.CsrMatrix.from_binary64(len(rp) - 1, rp, ci, v, None, P)
    crp, cci, cvr, cvi = problems.helmholtz7(4, 7)[:4]
    C = pkg.CsrMatrix.from_binary64(len(crp) - 1, crp, cci, cvr, cvi, P)
    return A, C, P


@pytest.mark.parametrize("k", [2, 3])
def test_build_problem_bitwise(k):
    import paper_2504_14498_b200 as pkg
    from paper_2504_14498_b200.grid import build_problem

    g = golden("grid_small.npz")
    A, C, P = _mats(pkg, k)
    pr = build_problem(A, P, "cd5_8")
    assert bits_equal(pr.x_star.re, g[f"r{k}_xstar"]) and bits_equal(pr.b.re, g[f"r{k}_b"])
    pc = build_problem(C, P, "helm4")
    assert bits_equal(pc.x_star.re, g[f"c{k}_xstar_re"])
    assert bits_equal(pc.x_star.im, g[f"c{k}_xstar_im"])
    assert bits_equal(pc.b.re, g[f"c{k}_b_re"]) and bits_equal(pc.b.im, g[f"c{k}_b_im"])


def test_default_grid_matches_reference():
    import paper_2504_14498_b200 as pkg
    from paper_2504_14498_b200.grid import (build_problem, default_grid, emit_report,
                                            parse_report, ratio_rows, run_benchmark)

    g = golden("grid_small.npz")
    A, _, P = _mats(pkg, 2)
    pr = build_problem(A, P, "cd5_8")
    suite = [(A, pr, pkg.SolverConfig(method=m, precision=p, precond=pre, spmv_mode=mode,
                                      eps_rel=1e-20))
             for m, p, pre, mode in default_grid(precisions=[P])]
    with pkg.reduction_mode("sequential"):
        rows = run_benchmark(suite)
    keys = [f"{r.method}|{r.precond}|{r.spmv_mode}" for r in rows]
    assert keys == list(g["grid_keys"])
    assert [r.iterations for r in rows] == list(g["grid_iterations"])
    assert [r.converged for r in rows] == list(g["grid_converged"])
    # twin-mode reductions: the reference's computation, so its residual and
    # error norms (GPBiCG's ilu0-mixed true residual included) are reproduced
    assert np.array_equal(np.array([r.true_relres for r in rows]), g["grid_true_relres"])
    assert np.array_equal(np.array([r.err2 for r in rows]), g["grid_err2"])
    text = emit_report(rows, "csv", ratios=True)
    assert parse_report(text) == rows
    rr = ratio_rows(rows)
    assert len(rr) == 4 and all(np.isfinite(x.ilu0_over_ilu0d) for x in rr)


def test_run_benchmark_jobs_pool_and_signature():
    """run_benchmark(suite, jobs, log) as the reference's (bench.py:179-216):
    a thread pool gives the same rows (timing fields aside); a failing cell
    becomes a non-converged row and is logged."""
    import paper_2504_14498_b200 as pkg
    from paper_2504_14498_b200.grid import build_problem, default_grid, run_benchmark, run_cell

    A, _, P = _mats(pkg, 2)
    pr = build_problem(A, P, "cd5_8")
    suite = [(A, pr, pkg.SolverConfig(method=m, precision=p, precond=pre, spmv_mode=mode,
                                      eps_rel=1e-20))
             for m, p, pre, mode in default_grid(methods=["bicgstab", "cgs"], precisions=[P])]
    lines = []
    one = run_benchmark(suite, 1, lines.append)
    pool = run_benchmark(suite, 4)  # second positional argument is `jobs`
    stable = lambda r: (r.matrix, r.method, r.precision, r.precond, r.spmv_mode, r.iterations,
                        r.converged, r.true_relres, r.err2)
    assert [stable(r) for r in pool] == [stable(r) for r in one]
    assert len(lines) == len(suite)
    row = run_cell(A, pr, suite[0][2], parallel_spmv=True)
    assert stable(row) == stable(one[0])
    wrong = pkg.DenseVector.zeros(A.n, pkg.Precision.TD, "real")  # precision mismatch
    bad_pr = type(pr)(pr.matrix_name, pr.field, pr.n, pr.x_star, wrong)
    failed = run_benchmark([(A, bad_pr, suite[0][2])], jobs=2, log=lines.append)
    assert failed[0].iterations == 0 and not failed[0].converged
    assert any(s.startswith("cell failed") for s in lines)
