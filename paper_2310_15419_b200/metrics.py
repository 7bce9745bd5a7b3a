"""Host-side metric and roofline arithmetic (no GPU, no oracle).

``gflops`` is the paper's and BASELINE.json's metric, 2·d·nnz(A)/t (PAPER.md:714-733,
Table tab:parallel, reproduces every printed GFlops; see tests/golden/paper_tab_parallel.csv).
"""
from __future__ import annotations


def gflops(d: int, nnz: int, seconds: float) -> float:
    """Sketch throughput 2·d·nnz(A)/t in GFLOP/s."""
    return 2.0 * float(d) * float(nnz) / float(seconds) / 1e9


def expected_nonzero_rows(m1: int, n1: int, rho: float) -> float:
    """E[Y] = m1 (1 - (1 - rho)^n1): expected number of rows of an m1 x n1 block with at
    least one nonzero when entries are nonzero with probability rho (
    the garbled PAPER.md:367 variant is not used, reading R13)."""
    return m1 * (1.0 - (1.0 - rho) ** n1)


def algorithmic_bytes(d: int, n: int, nnz: int, value_bytes: int) -> int:
    """Bytes the sketch must move at minimum: A read once (colptr int64, rowidx int32,
    values) plus Â written once."""
    return 8 * (n + 1) + 4 * nnz + value_bytes * nnz + value_bytes * d * n
