"""SAP least squares on the GPU: sketch with the fused kernel, QR, LSQR.
Synthetic tall sparse problems shaped like the paper's rail2586 (923269 x 2586, 8.0M nonzeros).

    python scripts/sap_demo.py [--m 1000000 --n 1000 --nnz 40 --dist gaussian --method qr]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2310_15419_b200 import sap  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=923_269)
    ap.add_argument("--n", type=int, default=2586)
    ap.add_argument("--nnz", type=int, default=3098)
    ap.add_argument("--decades", type=float, default=2.0)
    ap.add_argument("--dist", default="gaussian")
    ap.add_argument("--method", default="qr")
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    A, b = workloads.ls_problem(a.m, a.n, a.nnz, seed=1, col_scale_decades=a.decades)
    dev = torch.device("cuda:0")
    cp, ri, va = (torch.from_numpy(x).to(dev) for x in (A.colptr, A.rowidx, A.vals))
    bb = torch.from_numpy(b).to(dev)
    for rep in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = sap.sap_solve(cp, ri, va, A.m, A.n, bb, d=2 * A.n, seed=7, dist=a.dist, method=a.method)
        torch.cuda.synchronize()
        total = time.perf_counter() - t0
    print(json.dumps({"m": A.m, "n": A.n, "nnz": A.nnz, "d": 2 * A.n, "dist": a.dist, "method": a.method,
                      "iterations": res.iterations, "istop": res.istop, "error": res.error, "rank": res.rank,
                      "total_s": total, **res.times}))


if __name__ == "__main__":
    main()
