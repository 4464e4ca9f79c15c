"""Seeded synthetic inputs for the five BASELINE.json configurations.

The paper's SuiteSparse matrices are not available (no network), so these
generators stand in for them with the shapes, sizes and value
distributions BASELINE.json names.  All matrices
are binary64 CSR with int64 indices and strictly increasing columns per
row, i.e. exactly what ``CsrMatrix(..., Precision.F64)`` /
``CsrMatrix.demoted()`` holds in the reference (sparse.py:192-249).

Every generator is deterministic: the RNG draw order is fixed and
duplicates are summed left to right in binary64, so the CPU oracle, the
reference and the device path all see bit-identical inputs.  The right-hand
side is returned in binary64 form (``x_true`` for b = A x_true, or ``b64``
for a directly given b); the caller forms b in working precision with its
own SpMV, as the reference bench does (bench.py:88-104).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Problem",
    "convdiff5",
    "random_nonsym",
    "helmholtz7",
    "convdiff9",
    "cfg1",
    "cfg2",
    "cfg3",
    "cfg4",
    "cfg5",
    "CONFIGS",
]


@dataclass
class Problem:
    name: str
    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    val_re: np.ndarray
    val_im: np.ndarray | None = None
    x_true: np.ndarray | None = None  # b = A x_true (binary64 x)
    b64: np.ndarray | None = None  # b given directly (promoted exactly)
    methods: tuple = ()
    precisions: tuple = ()
    eps_rel: float = 1e-13
    eps_abs: float = 1e-100
    max_iter: int | None = None
    meta: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def field(self) -> str:
        return "real" if self.val_im is None else "complex"

    def checksum(self) -> str:
        import hashlib

        h = hashlib.sha256()
        for a in (self.row_ptr, self.col_idx, self.val_re, self.val_im,
                  self.x_true, self.b64):
            if a is not None:
                h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()


def _csr_from_sorted(n, rows, cols, vre, vim=None):
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    return row_ptr, cols.astype(np.int64), vre, vim


def convdiff5(m: int, pe: float) -> tuple:
    """2D upwind convection-diffusion, 5-point stencil on an m x m interior
    grid, h = 1/(m+1): (-u_xx - u_yy + Pe (u_x + u_y)) h^2 with backward
    differences -> centre 4 + 2 Pe h, W/S -(1 + Pe h), E/N -1 (natural
    ordering i = y*m + x, columns ascending S, W, C, E, N)."""
    h = 1.0 / (m + 1)
    c = 4.0 + 2.0 * pe * h
    ws = -(1.0 + pe * h)
    en = -1.0
    n = m * m
    idx = np.arange(n, dtype=np.int64)
    x = idx % m
    y = idx // m
    offs = [(-m, ws, y > 0), (-1, ws, x > 0), (0, c, np.ones(n, bool)),
            (1, en, x < m - 1), (m, en, y < m - 1)]
    rows, cols, vals = [], [], []
    for d, v, mask in offs:
        r = idx[mask]
        rows.append(r)
        cols.append(r + d)
        vals.append(np.full(r.size, v))
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    vals = np.concatenate(vals)
    order = np.lexsort((cols, rows))
    return _csr_from_sorted(n, rows[order], cols[order], vals[order])


def convdiff9(m: int, pe: float) -> tuple:
    """2D convection-diffusion, 9-point stencil on an m x m grid: compact
    (Mehrstellen) 9-point Laplacian [20, -4 edges, -1 corners]/(6h^2) plus
    backward-difference convection Pe (u_x + u_y), all scaled by 6h^2:
    centre 20 + 12 Pe h, W/S -4 - 6 Pe h, E/N -4, corners -1."""
    h = 1.0 / (m + 1)
    c = 20.0 + 12.0 * pe * h
    ws = -4.0 - 6.0 * pe * h
    en = -4.0
    co = -1.0
    n = m * m
    idx = np.arange(n, dtype=np.int64)
    x = idx % m
    y = idx // m
    offs = [
        (-m - 1, co, (y > 0) & (x > 0)),
        (-m, ws, y > 0),
        (-m + 1, co, (y > 0) & (x < m - 1)),
        (-1, ws, x > 0),
        (0, c, None),
        (1, en, x < m - 1),
        (m - 1, co, (y < m - 1) & (x > 0)),
        (m, en, y < m - 1),
        (m + 1, co, (y < m - 1) & (x < m - 1)),
    ]
    # rows are emitted in ascending column order per row by construction:
    # build a dense (n, 9) table and compress the valid entries row-major.
    colt = np.empty((n, 9), dtype=np.int64)
    valt = np.empty((n, 9))
    okt = np.empty((n, 9), dtype=bool)
    for t, (d, v, mask) in enumerate(offs):
        colt[:, t] = idx + d
        valt[:, t] = v
        okt[:, t] = True if mask is None else mask
    counts = okt.sum(axis=1)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    row_ptr[1:] = np.cumsum(counts)
    return row_ptr, colt[okt], valt[okt], None


def random_nonsym(n: int, d: int, seed: int) -> tuple:
    """Random nonsymmetric matrix: d off-diagonal draws per row at uniform
    columns (self hits dropped, duplicates summed left to right), N(0,1)
    values, diagonal 1.05 x the row's off-diagonal |.| sum with a random
    sign; x_true ~ U(-1, 1).  Draw order: cols, vals, signs, x_true."""
    rng = np.random.default_rng(seed)
    rows = np.repeat(np.arange(n, dtype=np.int64), d)
    cols = rng.integers(0, n, size=n * d, dtype=np.int64)
    vals = rng.standard_normal(n * d)
    signs = np.where(rng.integers(0, 2, size=n) == 0, -1.0, 1.0)
    x_true = rng.uniform(-1.0, 1.0, size=n)
    keep = cols != rows
    rows, cols, vals = rows[keep], cols[keep], vals[keep]
    key = rows * n + cols
    order = np.argsort(key, kind="stable")
    key, rows, cols, vals = key[order], rows[order], cols[order], vals[order]
    uniq, start, cnt = np.unique(key, return_index=True, return_counts=True)
    out = vals[start].copy()
    for g in np.nonzero(cnt > 1)[0]:
        s = 0.0
        for p in range(start[g], start[g] + cnt[g]):
            s = s + float(vals[p])
        out[g] = s
    orow = rows[start]
    ocol = cols[start]
    # np.bincount accumulates each bin sequentially in input order
    absum = np.bincount(orow, weights=np.abs(out), minlength=n)
    diag = 1.05 * absum * signs
    allr = np.concatenate([orow, np.arange(n, dtype=np.int64)])
    allc = np.concatenate([ocol, np.arange(n, dtype=np.int64)])
    allv = np.concatenate([out, diag])
    o = np.lexsort((allc, allr))
    rp, ci, vr, _ = _csr_from_sorted(n, allr[o], allc[o], allv[o])
    return rp, ci, vr, x_true


def helmholtz7(m: int, seed: int) -> tuple:
    """Complex shifted 3D 7-point Laplacian on an m^3 grid, h = 1/(m+1):
    A = h^-2 (L7 - (0.5 + 0.05i) I), L7 = 6 on the diagonal, -1 off it
    (SURVEY.md H7 natural reading).  b = U(-1,1) + i U(-1,1)."""
    n = m ** 3
    ih2 = float((m + 1) ** 2)
    dre = 5.5 * ih2
    dim = -0.05 * ih2
    off = -ih2
    idx = np.arange(n, dtype=np.int64)
    x = idx % m
    y = (idx // m) % m
    z = idx // (m * m)
    offs = [(-m * m, z > 0), (-m, y > 0), (-1, x > 0), (0, None), (1, x < m - 1),
            (m, y < m - 1), (m * m, z < m - 1)]
    colt = np.empty((n, 7), dtype=np.int64)
    ret = np.empty((n, 7))
    imt = np.zeros((n, 7))
    okt = np.empty((n, 7), dtype=bool)
    for t, (dd, mask) in enumerate(offs):
        colt[:, t] = idx + dd
        ret[:, t] = dre if dd == 0 else off
        if dd == 0:
            imt[:, t] = dim
        okt[:, t] = True if mask is None else mask
    counts = okt.sum(axis=1)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    row_ptr[1:] = np.cumsum(counts)
    rng = np.random.default_rng(seed)
    bre = rng.uniform(-1.0, 1.0, size=n)
    bim = rng.uniform(-1.0, 1.0, size=n)
    return row_ptr, colt[okt], ret[okt], imt[okt], bre + 1j * bim


def cfg1() -> Problem:
    rp, ci, v, _ = convdiff5(64, 10.0)
    n = 64 * 64
    return Problem("cfg1", n, rp, ci, v, x_true=np.ones(n),
                   methods=("bicgstab",), precisions=("dd",), eps_rel=1e-20,
                   max_iter=2000)


def cfg2(seed: int = 2) -> Problem:
    n = 20000
    rp, ci, v, xt = random_nonsym(n, 12, seed)
    return Problem("cfg2", n, rp, ci, v, x_true=xt,
                   methods=("bicg", "cgs", "bicgstab", "gpbicg"),
                   precisions=("td", "qd"), eps_rel=1e-30, max_iter=2000,
                   meta={"seed": seed})


def cfg3(m: int = 48, seed: int = 3) -> Problem:
    rp, ci, vr, vi, b = helmholtz7(m, seed)
    return Problem("cfg3", m ** 3, rp, ci, vr, vi, b64=b,
                   methods=("gpbicg", "bicgstab"), precisions=("dd",),
                   eps_rel=1e-24, meta={"seed": seed, "m": m})


def cfg4(m: int = 2048) -> Problem:
    rp, ci, v, _ = convdiff9(m, 5.0)
    n = m * m
    return Problem("cfg4", n, rp, ci, v, x_true=np.ones(n),
                   methods=("bicgstab",), precisions=("dd",), eps_rel=1e-300,
                   eps_abs=1e-300, max_iter=200, meta={"m": m})


def cfg5(system: int, base_seed: int = 5000, n: int = 50000) -> Problem:
    rp, ci, v, xt = random_nonsym(n, 16, base_seed + system)
    return Problem(f"cfg5[{system}]", n, rp, ci, v, x_true=xt,
                   methods=("cgs", "bicgstab"), precisions=("qd",),
                   eps_rel=1e-40, max_iter=2000,
                   meta={"seed": base_seed + system, "system": system})


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5}
