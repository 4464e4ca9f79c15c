"""Benchmark grid and report emission (reference
bench.py:44-309): schema, CSV/JSON emission, CSV round trip and Table-4
ratio rows on synthetic rows (CPU); the device grid itself is checked in
tests/test_gpu_grid.py."""

from __future__ import annotations

import io
import json
import math

import pytest

from paper_2504_14498_b200.grid import (CSV_HEADER, BenchRow, default_grid, emit_report,
                                        parse_report, ratio_rows)
from paper_2504_14498_b200 import Precision, PrecondMode


def _rows():
    out = []
    for m in ("bicg", "cgs"):
        for pre, mode, ms in (("none", "full", 2.0), ("ilu0", "full", 6.0),
                              ("none", "mixed", 1.0), ("ilu0-mixed", "mixed", 1.5)):
            out.append(BenchRow("m1", m, "DD", pre, mode, 10, True, 0.1, ms, 1e-21, 1e-19))
    return out


def test_schema_and_grid():
    assert CSV_HEADER == ["matrix", "method", "precision", "precond", "spmv_mode",
                          "iterations", "converged", "total_s", "ms_per_iter",
                          "true_relres", "err2"]
    g = default_grid()
    assert len(g) == 4 * 3 * 4
    assert g[0] == ("bicg", Precision.DD, PrecondMode.NONE, "full")
    assert g[3] == ("bicg", Precision.DD, PrecondMode.ILU0_MIXED, "mixed")


def test_csv_round_trip_and_ratios():
    rows = _rows()
    buf = io.StringIO()
    text = emit_report(rows, "csv", out=buf, ratios=True)
    assert buf.getvalue() == text
    back = parse_report(text)
    assert back == rows
    rr = ratio_rows(rows)
    assert len(rr) == 2
    assert rr[0].ilu0_over_plain == 3.0 and rr[0].ilu0d_over_plaind == 1.5
    assert rr[0].ilu0_over_ilu0d == 4.0
    assert "ilu0_over_ilu0d" in text.splitlines()[len(rows) + 2]


def test_json_and_errors():
    rows = _rows()
    d = json.loads(emit_report(rows, "json", ratios=True))
    assert len(d["rows"]) == len(rows) and len(d["ratios"]) == 2
    with pytest.raises(ValueError):
        emit_report([], "csv")
    with pytest.raises(ValueError):
        emit_report(rows, "xml")
    with pytest.raises(ValueError):
        parse_report("a,b\n")
    nan_rows = [BenchRow("m", "bicg", "DD", "ilu0", "full", 0, False, math.nan, math.nan,
                         math.nan, math.nan)]
    assert math.isnan(ratio_rows(nan_rows)[0].ilu0_over_plain)
