"""Tensor-core (sk_rad_f4_kernel) vs SIMT (sk_rad_kernel<double>) time per column length L: the
measurement behind the plan's shortest tensor-core column (SKETCH_F4_MIN_COL, sketch_api.cu).

    SKETCH_F4_MIN_COL=1 python scripts/f4_threshold_sweep.py [--d 2000] [--nnz 8000000]

Each matrix has nnz / L columns of exactly L nonzeros (uniform rows, N(0,1) values, m = 5e6), d rows of Â.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2310_15419_b200 import sketch as sk  # noqa: E402


def time_path(path, A, d, reps=5):
    sk.set_rad_f64_path(path)
    dev = torch.device("cuda:0")
    plan = sk.Plan(torch.from_numpy(A.colptr).to(dev), torch.from_numpy(A.rowidx).to(dev), d, A.m, "f64")
    vals = torch.from_numpy(A.vals).to(dev)
    out = torch.empty((A.n, d), dtype=torch.float64, device=dev)
    for _ in range(2):
        plan.apply(vals, 1, "rademacher", out=out)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
    for r in range(reps):
        ev[2 * r].record()
        plan.apply(vals, 1, "rademacher", out=out)
        ev[2 * r + 1].record()
    torch.cuda.synchronize()
    name = plan.kernel_name("rademacher")
    plan.close()
    return float(np.median([ev[2 * r].elapsed_time(ev[2 * r + 1]) for r in range(reps)])), name


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=2000)
    ap.add_argument("--nnz", type=int, default=8_000_000)
    a = ap.parse_args()
    for L in (64, 128, 256, 384, 512, 768, 1024, 1536, 2048, 4096, 16384):
        n = max(1, a.nnz // L)
        A = workloads.random_csc(5_000_000, n, L, seed=L)
        t4, n4 = time_path("fp4", A, a.d)
        ts, ns = time_path("simt", A, a.d)
        e = 2.0 * a.d * A.nnz
        print(f"L {L:6d} n {n:6d}  fp4 {t4:8.3f} ms ({e / t4 / 1e9:8.0f} TF/s, {n4.split(' ')[0]})  "
              f"simt {ts:8.3f} ms ({e / ts / 1e9:8.0f} TF/s)  fp4/simt {t4 / ts:.3f}", flush=True)
    sk.set_rad_f64_path("fp4")


if __name__ == "__main__":
    main()
