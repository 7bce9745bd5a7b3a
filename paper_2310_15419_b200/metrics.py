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


# ---------------------------------------------------------------- roofline
#
# T_roof = max(T_HBM, T_FP, T_INT) for one sketch of a d x m S with A (n columns, nnz stored
# entries, nnzrows nonzero rows):
#   T_HBM = algorithmic bytes (A read once, Â written once) / measured HBM bandwidth;
#   T_FP  = (d nnz + X G) / (SMs x lanes x clock): one fused multiply-add per (row of Â, nonzero) plus
#           X FP operations per Philox block for the entry transform, on the FP64 (64 lanes/SM) or
#           FP32 (128 lanes/SM) pipe of the arithmetic dtype;
#   T_INT = G / measured Philox4x32-10 rate;
#   G     = ceil(d / E) nnzrows: every needed S entry generated ONCE (Algorithm 4's ideal with
#           b_n = n) -- the strict count; ceil(d / E) nnz (Algorithm 3's
#           regeneration per stored nonzero) is reported beside it as a diagnostic.
# The per-pipe rates below are frozen measurements (profiles/r01_microbench.json, B200 at
# 1965 MHz, scripts/microbench.cu): Philox blocks/s of a Philox-only loop, and the FP64 operations a
# Box-Muller pair costs beyond its two multiply-adds in the r01 kernel (ncu instruction mix).
PHILOX_BLOCKS_PER_S = 4.549e11
ENTRIES_PER_BLOCK = {"rademacher": 128, "uniform": 2, "gaussian": 2, "uniform24": 4}
FP_OPS_PER_BLOCK = {"rademacher": 0, "uniform": 2, "gaussian": 38, "uniform24": 4}
N_SMS = 148


def fp_lane_rate(dtype: str, sm_mhz: float) -> float:
    """FP lane-operations per second of the dtype's pipe: 148 SMs x {64 fp64, 128 fp32} lanes x clock."""
    return N_SMS * (64 if dtype == "f64" else 128) * sm_mhz * 1e6


def roofline(dist: str, dtype: str, d: int, n: int, nnz: int, nnzrows: int, hbm_gbs: float,
             sm_mhz: float) -> dict:
    """The strict roofline of one sketch (times in seconds); bound names the slowest term."""
    w = 8 if dtype == "f64" else 4
    E = ENTRIES_PER_BLOCK[dist]
    g_strict = -(-d // E) * nnzrows
    g_alg3 = -(-d // E) * nnz
    by = algorithmic_bytes(d, n, nnz, w)
    t_hbm = by / (hbm_gbs * 1e9)
    t_fp = (float(d) * nnz + FP_OPS_PER_BLOCK[dist] * g_strict) / fp_lane_rate(dtype, sm_mhz)
    t_int = g_strict / PHILOX_BLOCKS_PER_S
    terms = {"hbm": t_hbm, ("fp64_pipe" if dtype == "f64" else "fp32_pipe"): t_fp, "int_philox": t_int}
    bound = max(terms, key=terms.get)
    return {"bound": bound, "t_roof": terms[bound], "t_hbm": t_hbm, "t_fp": t_fp, "t_int": t_int,
            "algorithmic_bytes": by, "g_calls_strict": g_strict, "g_calls_alg3": g_alg3,
            "fp_ops": float(d) * nnz + FP_OPS_PER_BLOCK[dist] * g_strict}


def roofline_report(rl: dict, t_kernel: float, dtype: str, hbm_gbs: float, sm_mhz: float) -> dict:
    """achieved / peak / frac of the bound term for a kernel that took t_kernel seconds."""
    b = rl["bound"]
    if b == "hbm":
        ach, peak, unit = rl["algorithmic_bytes"] / t_kernel / 1e9, hbm_gbs, "GB/s"
    elif b == "int_philox":
        ach, peak, unit = rl["g_calls_strict"] / t_kernel / 1e9, PHILOX_BLOCKS_PER_S / 1e9, "Gblocks/s"
    else:   # FP pipe, counted as 2 flop per lane-op (the metric's flop per multiply-add)
        ach, peak, unit = 2 * rl["fp_ops"] / t_kernel / 1e12, 2 * fp_lane_rate(dtype, sm_mhz) / 1e12, "TFLOP/s"
    return {"bound": b, "achieved": ach, "peak": peak, "unit": unit, "frac": rl["t_roof"] / t_kernel,
            "t_roof_ms": rl["t_roof"] * 1e3}
