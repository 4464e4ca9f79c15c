"""Matrix Market ingestion: the data format on the input
side of the hot path, so the paper's SuiteSparse matrices can be solved when
fixtures are supplied.

Same entry points and semantics as the reference (sparse.py:47-189, 275-338):
``parse_matrix_market(text_or_file) -> CooMatrix`` (coordinate layout only;
fields real / integer / complex / pattern; symmetries general / symmetric /
hermitian / skew-symmetric, stored once with the tag kept; 0-based indices;
``MatrixMarketError`` with the offending line number), ``read_matrix_market``
and ``coo_to_csr(coo, precision) -> CsrMatrix`` (square only; symmetric
mirror entries, hermitian conjugated, skew negated; rows sorted, then
columns; duplicates summed exactly in MC arithmetic in file order after a
stable (row, col) sort -- the host MC add is the device twin of
``_mccore.mc_add``, so the sums are the reference's bit for bit).
Host-side code: ingestion runs once per matrix, before the device upload.
"""

from __future__ import annotations

import io
from dataclasses import dataclass

import numpy as np

from .multicomponent import Precision, add_limbs
from .sparse import CsrMatrix

__all__ = ["MatrixMarketError", "CooMatrix", "parse_matrix_market",
           "read_matrix_market", "coo_to_csr"]

SYMMETRIES = ("general", "symmetric", "hermitian", "skew-symmetric")
FIELDS = ("real", "integer", "complex", "pattern")


class MatrixMarketError(ValueError):
    """Malformed Matrix Market input; ``line`` is the 1-based line number."""

    def __init__(self, message: str, line: int | None = None):
        self.line = line
        super().__init__(message if line is None else f"line {line}: {message}")


@dataclass
class CooMatrix:
    n_rows: int
    n_cols: int
    row: np.ndarray
    col: np.ndarray
    val_re: np.ndarray
    val_im: np.ndarray | None
    symmetry: str = "general"

    @property
    def field(self) -> str:
        return "complex" if self.val_im is not None else "real"

    @property
    def nnz(self) -> int:
        return int(self.row.shape[0])


def _header(line: str):
    if not line.startswith("%%MatrixMarket"):
        raise MatrixMarketError("missing %%MatrixMarket header", 1)
    tok = [t.lower() for t in line.split()]
    if len(tok) != 5:
        raise MatrixMarketError(f"header must have 5 tokens, got {len(tok)}", 1)
    _, obj, layout, field, sym = tok
    if obj != "matrix":
        raise MatrixMarketError(f"unsupported object {obj!r}", 1)
    if layout != "coordinate":
        raise MatrixMarketError(
            f"unsupported layout {layout!r} (only 'coordinate' is supported)", 1)
    if field not in FIELDS:
        raise MatrixMarketError(f"unknown field {field!r}", 1)
    if sym not in SYMMETRIES:
        raise MatrixMarketError(f"unknown symmetry {sym!r}", 1)
    return field, sym


def parse_matrix_market(source) -> CooMatrix:
    """Coordinate Matrix Market text (a string or a text file object)."""
    lines = io.StringIO(source) if isinstance(source, str) else source
    field, sym = _header(lines.readline())
    ln = 1
    size = None
    for raw in lines:
        ln += 1
        s = raw.strip()
        if s and not s.startswith("%"):
            size = s
            break
    if size is None:
        raise MatrixMarketError("missing size line", ln + 1)
    tok = size.split()
    if len(tok) != 3:
        raise MatrixMarketError(f"size line must be 'rows cols nnz', got {size!r}", ln)
    try:
        nr, nc, nnz = (int(t) for t in tok)
    except ValueError as exc:
        raise MatrixMarketError(f"bad size line {size!r}", ln) from exc
    if nr <= 0 or nc <= 0 or nnz < 0:
        raise MatrixMarketError("rows, cols must be positive and nnz >= 0", ln)
    nval = {"pattern": 0, "complex": 2}.get(field, 1)
    row = np.empty(nnz, np.int64)
    col = np.empty(nnz, np.int64)
    vre = np.empty(nnz, np.float64)
    vim = np.empty(nnz, np.float64) if field == "complex" else None
    m = 0
    for raw in lines:
        ln += 1
        s = raw.strip()
        if not s or s.startswith("%"):
            continue
        if m >= nnz:
            raise MatrixMarketError(f"more than the declared {nnz} entries", ln)
        tok = s.split()
        try:
            i, j = int(tok[0]), int(tok[1])
        except (ValueError, IndexError) as exc:
            raise MatrixMarketError(f"bad entry {s!r}", ln) from exc
        if not (1 <= i <= nr and 1 <= j <= nc):
            raise MatrixMarketError(f"index ({i}, {j}) out of bounds for {nr}x{nc}", ln)
        if len(tok) != 2 + nval:
            raise MatrixMarketError(f"bad value fields for {field} entry {s!r}", ln)
        try:
            re_v = float(tok[2]) if nval else 1.0
            im_v = float(tok[3]) if nval == 2 else 0.0
        except ValueError as exc:
            raise MatrixMarketError(f"bad value fields for {field} entry {s!r}", ln) from exc
        if not (np.isfinite(re_v) and np.isfinite(im_v)):
            raise MatrixMarketError(f"non-finite value in {s!r}", ln)
        row[m], col[m], vre[m] = i - 1, j - 1, re_v
        if vim is not None:
            vim[m] = im_v
        m += 1
    if m != nnz:
        raise MatrixMarketError(f"declared {nnz} entries but found {m}", ln)
    return CooMatrix(nr, nc, row, col, vre, vim, sym)


def read_matrix_market(path) -> CooMatrix:
    with open(path, "r", encoding="ascii", errors="replace") as fh:
        return parse_matrix_market(fh)


def coo_to_csr(coo: CooMatrix, precision: Precision) -> CsrMatrix:
    """Square CSR at ``precision`` (see the module docstring)."""
    if coo.n_rows != coo.n_cols:
        raise ValueError(f"matrix must be square, got {coo.n_rows}x{coo.n_cols}")
    n, k = coo.n_rows, precision.k
    r, c, vr = coo.row, coo.col, coo.val_re
    vi = coo.val_im if coo.val_im is not None else np.zeros_like(vr)
    if coo.symmetry != "general":
        off = r != c
        mir_re, mir_im = vr[off].copy(), vi[off].copy()
        if coo.symmetry == "hermitian":
            mir_im = -mir_im
        elif coo.symmetry == "skew-symmetric":
            mir_re, mir_im = -mir_re, -mir_im
        r, c = np.concatenate([r, c[off]]), np.concatenate([c, coo.row[off]])
        vr, vi = np.concatenate([vr, mir_re]), np.concatenate([vi, mir_im])
    order = np.lexsort((c, r))  # stable: duplicates keep file order
    r, c, vr, vi = r[order], c[order], vr[order], vi[order]
    key = r * n + c
    first = np.flatnonzero(np.r_[True, key[1:] != key[:-1]]) if len(key) else \
        np.zeros(0, np.int64)
    ends = np.r_[first[1:], len(key)]
    nnz = len(first)
    out_re = np.zeros((nnz, k))
    out_im = np.zeros((nnz, k))
    single = ends - first == 1
    out_re[single, 0] = vr[first[single]]
    out_im[single, 0] = vi[first[single]]
    pad = (0.0,) * (k - 1)
    for t in np.flatnonzero(~single):  # exact MC sums of the duplicates
        sr = si = (0.0,) * k
        for q in range(first[t], ends[t]):
            if k == 1:
                sr, si = (sr[0] + vr[q],), (si[0] + vi[q],)
            else:
                sr = add_limbs(sr, (float(vr[q]),) + pad)
                si = add_limbs(si, (float(vi[q]),) + pad)
        out_re[t], out_im[t] = sr, si
    row_ptr = np.zeros(n + 1, np.int64)
    np.add.at(row_ptr, r[first] + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    return CsrMatrix(n, row_ptr, c[first].astype(np.int64), np.ascontiguousarray(out_re),
                     np.ascontiguousarray(out_im) if coo.field == "complex" else None,
                     precision)
