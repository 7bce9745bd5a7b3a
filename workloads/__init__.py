"""Seeded synthetic inputs A (tall sparse CSC) for the sketch Â = S·A.

This module holds NONE of the method's arithmetic (no RNG for S, no transforms, no
products): it only draws the sparse matrices A that both the CUDA path and the CPU oracle
consume, so it is the one module the two sides share (DESIGN.md §"Inputs").

The five configurations are BASELINE.json ``configs[0..4]`` (c1..c5).  They stand in for
the paper's SuiteSparse test matrices (Table ``matrix:name``) and its
"tall sparse least-squares inputs", which are not available here.
Recipes (DESIGN.md §"Inputs"):

  c1  m=1e5,  n=500,  d=1000  : 20 distinct uniform rows per column, vals N(0,1) fp64; ±1, seed 0
  c2  m=1e6,  n=1000, d=2000  : 1000 distinct uniform rows per column, vals U(-1,1) fp64; uniform, seed 1
  c3  m=4e6,  n=2000, d=6000  : column lengths L ~ p(L) ∝ L^-1.5 on [10, 20000] (inverse CDF + floor,
                                DESIGN.md reading R17 "A"), distinct uniform rows, vals N(0,1); Gaussian, seed 2
  c4  m=1e7,  n=5000, d=10000 : 400 distinct rows inside a random window of 1e5 rows, vals N(0,1)
                                rounded to fp32; ±1, seed 3
  c5  m=5e7,  n=1000, d=2000  : every row exactly one nonzero in a uniform column, vals N(0,1) fp64;
                                ±1, seed 4.  Generated in fixed row chunks with per-chunk seeds, so any
                                row shard [r0, r1) is produced identically and independently.

A's own generator is ``numpy.random.default_rng(1000 + c)`` (reading R19).
Rows within a column are sorted ascending and distinct (reading R18).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class CSC:
    """A tall sparse matrix in 0-based CSC form (int64 colptr, int32 rowidx)."""
    m: int
    n: int
    colptr: np.ndarray
    rowidx: np.ndarray
    vals: np.ndarray
    row_offset: int = 0          # global index of local row 0 (row shards)
    meta: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.rowidx.shape[0])

    def column(self, k: int):
        s, e = int(self.colptr[k]), int(self.colptr[k + 1])
        return self.rowidx[s:e], self.vals[s:e]

    def select_columns(self, cols) -> "CSC":
        """Sub-matrix A[:, cols] (cols in the given order)."""
        cols = np.asarray(cols, dtype=np.int64)
        lens = self.colptr[cols + 1] - self.colptr[cols]
        colptr = np.zeros(len(cols) + 1, dtype=np.int64)
        np.cumsum(lens, out=colptr[1:])
        idx = np.concatenate([np.arange(self.colptr[c], self.colptr[c + 1]) for c in cols]) \
            if len(cols) else np.zeros(0, dtype=np.int64)
        return CSC(self.m, len(cols), colptr, self.rowidx[idx], self.vals[idx],
                   self.row_offset, dict(self.meta))

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.m, self.n), dtype=np.float64)
        for k in range(self.n):
            r, v = self.column(k)
            np.add.at(out[:, k], r.astype(np.int64), v.astype(np.float64))
        return out


@dataclass(frozen=True)
class Config:
    name: str
    m: int
    n: int
    d: int
    dist: str
    seed: int
    dtype: str          # value dtype of A and of the kernel arithmetic ("f64" / "f32")
    note: str


CONFIGS = {
    "c1": Config("c1", 100_000, 500, 1000, "rademacher", 0, "f64",
                 "20 distinct uniform rows/column, vals N(0,1)"),
    "c2": Config("c2", 1_000_000, 1000, 2000, "uniform", 1, "f64",
                 "1000 distinct uniform rows/column, vals U(-1,1)"),
    "c3": Config("c3", 4_000_000, 2000, 6000, "gaussian", 2, "f64",
                 "power-law column lengths p(L)~L^-1.5 on [10,20000] (reading A), vals N(0,1)"),
    "c4": Config("c4", 10_000_000, 5000, 10000, "rademacher", 3, "f32",
                 "400 distinct rows in a random 1e5-row window per column, vals N(0,1) fp32"),
    "c5": Config("c5", 50_000_000, 1000, 2000, "rademacher", 4, "f64",
                 "one nonzero per row in a uniform column, vals N(0,1)"),
}

C5_CHUNK_ROWS = 1 << 20


def _finish(m, n, cols_of_nnz_lists, vals_lists, dtype, meta) -> CSC:
    lens = np.array([len(r) for r in cols_of_nnz_lists], dtype=np.int64)
    colptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=colptr[1:])
    rowidx = (np.concatenate(cols_of_nnz_lists) if n else np.zeros(0)).astype(np.int32)
    vals = (np.concatenate(vals_lists) if n else np.zeros(0)).astype(dtype)
    return CSC(m, n, colptr, rowidx, vals, 0, meta)


def _distinct_sorted(rng, lo: int, hi: int, k: int) -> np.ndarray:
    rows = rng.choice(hi - lo, size=k, replace=False) + lo
    rows.sort()
    return rows


def powerlaw_lengths(rng, n: int, alpha: float = 1.5, lmin: int = 10, lmax: int = 20000) -> np.ndarray:
    """L_k i.i.d. with density ∝ L^-alpha on [lmin, lmax], inverse CDF then floor."""
    u = rng.random(n)
    a1 = 1.0 - alpha
    lo, hi = lmin ** a1, lmax ** a1
    L = (lo + u * (hi - lo)) ** (1.0 / a1)
    return np.clip(np.floor(L).astype(np.int64), lmin, lmax)


def make_config(name: str, row_range=None) -> CSC:
    """A for config ``name`` (c1..c5).  ``row_range=(r0, r1)`` (c5 only) returns the row
    shard A[r0:r1, :] with local row indices and ``row_offset = r0``."""
    cfg = CONFIGS[name]
    c = int(name[1:])
    meta = {"config": name, "seed_A": 1000 + c}
    if name == "c5":
        return _make_c5(cfg, row_range, meta)
    if row_range is not None:
        raise ValueError("row_range is only supported for c5")
    rng = np.random.default_rng(1000 + c)
    rows_l, vals_l = [], []
    if name == "c1":
        for _ in range(cfg.n):
            rows_l.append(_distinct_sorted(rng, 0, cfg.m, 20))
            vals_l.append(rng.standard_normal(20))
        return _finish(cfg.m, cfg.n, rows_l, vals_l, np.float64, meta)
    if name == "c2":
        for _ in range(cfg.n):
            rows_l.append(_distinct_sorted(rng, 0, cfg.m, 1000))
            vals_l.append(rng.uniform(-1.0, 1.0, 1000))
        return _finish(cfg.m, cfg.n, rows_l, vals_l, np.float64, meta)
    if name == "c3":
        L = powerlaw_lengths(rng, cfg.n)
        for k in range(cfg.n):
            rows_l.append(_distinct_sorted(rng, 0, cfg.m, int(L[k])))
            vals_l.append(rng.standard_normal(int(L[k])))
        meta["reading"] = "R17-A (literal exponent 1.5 on [10, 20000]; realised nnz reported)"
        return _finish(cfg.m, cfg.n, rows_l, vals_l, np.float64, meta)
    if name == "c4":
        for _ in range(cfg.n):
            s = int(rng.integers(0, cfg.m - 100_000 + 1))
            rows_l.append(_distinct_sorted(rng, s, s + 100_000, 400))
            vals_l.append(rng.standard_normal(400))
        return _finish(cfg.m, cfg.n, rows_l, vals_l, np.float32, meta)
    raise KeyError(name)


def _c5_chunk(cfg: Config, ci: int, child_seeds):
    rng = np.random.default_rng(child_seeds[ci])
    r0 = ci * C5_CHUNK_ROWS
    cnt = min(C5_CHUNK_ROWS, cfg.m - r0)
    cols = rng.integers(0, cfg.n, size=cnt, dtype=np.int64)
    vals = rng.standard_normal(cnt)
    return cols, vals


def _make_c5(cfg: Config, row_range, meta) -> CSC:
    r0, r1 = (0, cfg.m) if row_range is None else (int(row_range[0]), int(row_range[1]))
    if not (0 <= r0 <= r1 <= cfg.m):
        raise ValueError("bad row range")
    nchunks = (cfg.m + C5_CHUNK_ROWS - 1) // C5_CHUNK_ROWS
    child = np.random.SeedSequence(1005).spawn(nchunks)
    cols_parts, vals_parts = [], []
    for ci in range(r0 // C5_CHUNK_ROWS, (r1 + C5_CHUNK_ROWS - 1) // C5_CHUNK_ROWS if r1 > r0 else 0):
        cols, vals = _c5_chunk(cfg, ci, child)
        base = ci * C5_CHUNK_ROWS
        a, b = max(r0, base) - base, min(r1, base + len(cols)) - base
        cols_parts.append(cols[a:b])
        vals_parts.append(vals[a:b])
    cols = np.concatenate(cols_parts) if cols_parts else np.zeros(0, dtype=np.int64)
    vals = np.concatenate(vals_parts) if vals_parts else np.zeros(0)
    return rows_by_column(r1 - r0, cfg.n, cols, vals, row_offset=r0, meta=meta)


def rows_by_column(m: int, n: int, col_of_row, vals_of_row, row_offset: int = 0, meta=None) -> CSC:
    """CSC of a matrix given as one (column, value) per local row, rows ascending per column."""
    col16 = np.asarray(col_of_row).astype(np.int16 if n < 32768 else np.int64)
    order = np.argsort(col16, kind="stable")       # stable: rows stay ascending within a column
    counts = np.bincount(np.asarray(col_of_row, dtype=np.int64), minlength=n)
    colptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=colptr[1:])
    rowidx = order.astype(np.int32)
    vals = np.asarray(vals_of_row, dtype=np.float64)[order]
    return CSC(m, n, colptr, rowidx, vals, row_offset, dict(meta or {}))


def shard_rows(m: int, world: int, rank: int):
    """Contiguous row shard [r_g, r_{g+1}) with r_g = floor(g*m/G)."""
    return (rank * m) // world, ((rank + 1) * m) // world


def shard_csc(A: CSC, world: int, rank: int) -> CSC:
    """Row shard of an in-memory CSC (local rows, row_offset advanced)."""
    r0, r1 = shard_rows(A.m, world, rank)
    cols = []
    vals = []
    keep_r = []
    for k in range(A.n):
        r, v = A.column(k)
        sel = (r >= r0) & (r < r1)
        keep_r.append((r[sel] - r0).astype(np.int32))
        vals.append(v[sel])
        cols.append(int(sel.sum()))
    colptr = np.zeros(A.n + 1, dtype=np.int64)
    np.cumsum(np.array(cols, dtype=np.int64), out=colptr[1:])
    rowidx = np.concatenate(keep_r) if A.n else np.zeros(0, dtype=np.int32)
    v = np.concatenate(vals) if A.n else np.zeros(0, dtype=A.vals.dtype)
    return CSC(r1 - r0, A.n, colptr, rowidx.astype(np.int32), v.astype(A.vals.dtype),
               A.row_offset + r0, dict(A.meta))


def col_slice(A: CSC, c0: int, c1: int) -> CSC:
    """Columns [c0, c1) of an in-memory CSC (all rows; colptr rebased to 0)."""
    p0, p1 = int(A.colptr[c0]), int(A.colptr[c1])
    meta = dict(A.meta)
    meta["col_range"] = (int(c0), int(c1))
    return CSC(A.m, c1 - c0, (A.colptr[c0:c1 + 1] - p0).astype(np.int64), A.rowidx[p0:p1].copy(),
               A.vals[p0:p1].copy(), A.row_offset, meta)


# ---------------------------------------------------------------- small / edge-case inputs

def random_csc(m: int, n: int, nnz_per_col, seed: int, dtype=np.float64, *, values="normal",
               sorted_rows=True, duplicates=False) -> CSC:
    """Random CSC with ``nnz_per_col`` (int or per-column list) entries per column."""
    rng = np.random.default_rng(seed)
    if np.isscalar(nnz_per_col):
        lens = [int(nnz_per_col)] * n
    else:
        lens = [int(x) for x in nnz_per_col]
    rows_l, vals_l = [], []
    for k in range(n):
        L = lens[k]
        if duplicates:
            r = rng.integers(0, m, size=L)
        else:
            r = rng.choice(m, size=min(L, m), replace=False)
        if sorted_rows:
            r = np.sort(r)
        if values == "normal":
            v = rng.standard_normal(len(r))
        elif values == "uniform":
            v = rng.uniform(-1, 1, len(r))
        elif values == "smallint":
            v = rng.integers(-8, 9, size=len(r)).astype(np.float64)
        else:
            raise ValueError(values)
        rows_l.append(r)
        vals_l.append(v)
    return _finish(m, n, rows_l, vals_l, dtype, {"seed_A": seed})


def abnormal(kind: str, m: int, n: int, nnz: int, seed: int) -> CSC:
    """Miniature 'exotic sparsity' patterns in the spirit of PAPER.md:679-707
    (Table tab:extreme_examples): 'A' = nonzeros packed into few dense rows,
    'B' = uniform scatter, 'C' = nonzeros packed into few dense columns."""
    rng = np.random.default_rng(seed)
    if kind == "A":
        nrows = max(1, nnz // n)
        rows = rng.choice(m, size=nrows, replace=False)
        rows.sort()
        lens = [nrows] * n
        rl = [rows.copy() for _ in range(n)]
    elif kind == "B":
        per = max(1, nnz // n)
        lens = [per] * n
        rl = [np.sort(rng.choice(m, size=per, replace=False)) for _ in range(n)]
    elif kind == "C":
        ncols = max(1, nnz // m) + 1
        lens = [0] * n
        rl = [np.zeros(0, dtype=np.int64) for _ in range(n)]
        for c in rng.choice(n, size=min(ncols, n), replace=False):
            per = min(m, nnz // ncols)
            rl[c] = np.sort(rng.choice(m, size=per, replace=False))
            lens[c] = per
    else:
        raise ValueError(kind)
    vl = [rng.standard_normal(len(r)) for r in rl]
    return _finish(m, n, rl, vl, np.float64, {"abnormal": kind})


def abnormal_paper(kind: str, m: int = 100_000, n: int = 10_000, seed: int = 0) -> CSC:
    """The exotic patterns of Table tab:extreme_examples as PAPER.md:699-701 describes them
    (m = 100000, n = 10000, density ~1e-3, N(0,1) values):
    'A': every 1000th row dense, all other rows zero;
    'B': ~2998/3000 of the nonzeros in the middle third of the columns (about 300 random rows per
         middle column), the rest one nonzero in random outer columns;
    'C': every 1000th column dense, all other columns zero."""
    rng = np.random.default_rng(seed)
    if kind == "A":
        rows = np.arange(0, m, 1000, dtype=np.int64)
        rl = [rows for _ in range(n)]
    elif kind == "B":
        total = int(round(1e-3 * m * n))
        mid0, mid1 = n // 3, (2 * n) // 3
        inner = int(round(total * 2998 / 3000))
        per, extra = divmod(inner, mid1 - mid0)
        rl = [np.zeros(0, dtype=np.int64) for _ in range(n)]
        for i, k in enumerate(range(mid0, mid1)):
            rl[k] = np.sort(rng.choice(m, size=per + (1 if i < extra else 0), replace=False))
        outer = np.array([k for k in range(n) if not mid0 <= k < mid1])
        for k in rng.choice(outer, size=min(total - inner, outer.size), replace=False):
            rl[k] = rng.integers(0, m, size=1)
    elif kind == "C":
        full = np.arange(m, dtype=np.int64)
        rl = [full if k % 1000 == 0 else np.zeros(0, dtype=np.int64) for k in range(n)]
    else:
        raise ValueError(kind)
    vl = [rng.standard_normal(len(r)) for r in rl]
    return _finish(m, n, rl, vl, np.float64, {"abnormal_paper": kind})


# ---------------------------------------------------------------- least-squares problems (SAP, §8(f) f2)

def ls_problem(m: int, n: int, nnz_per_col, seed: int, noise: float = 1.0, col_scale_decades: float = 0.0):
    """Synthetic tall sparse least-squares problem in the paper's recipe: A random
    CSC (N(0,1) values), b = A w + noise * N(0, I) with w ~ N(0, I).  col_scale_decades > 0 scales
    column k by 10^U(-c, c) (ill-conditioned A).  Stands in for the SuiteSparse matrices of Table
    matrix:name_extended, which are not available.  Returns (CSC, b)."""
    A = random_csc(m, n, nnz_per_col, seed=seed)
    rng = np.random.default_rng(seed + 7)
    if col_scale_decades > 0:
        sc = 10.0 ** rng.uniform(-col_scale_decades, col_scale_decades, size=n)
        A.vals = A.vals * np.repeat(sc, np.diff(A.colptr))
    w = rng.standard_normal(n)
    Aw = np.zeros(m)
    np.add.at(Aw, A.rowidx, A.vals * np.repeat(w, np.diff(A.colptr)))
    return A, Aw + noise * rng.standard_normal(m)
