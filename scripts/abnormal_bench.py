"""Algorithm 3 (kji) vs Algorithm 4 (jki) on the exotic sparsity patterns of Table
tab:extreme_examples: m = 100000, n = 10000, density 1e-3, S uniform(-1, 1).
Conversion (plan) time and compute (apply) time, like the paper's table.

    python scripts/abnormal_bench.py [--d 2000] [--dist uniform] [--reps 5]
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
from paper_2310_15419_b200 import sketch as sk  # noqa: E402


def timed_apply(plan, vals, dist, reps, seed=5):
    out = torch.empty((plan.n, plan.d), dtype=vals.dtype, device=vals.device)
    plan.apply(vals, seed, dist, out=out)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
    for r in range(reps):
        ev[2 * r].record()
        plan.apply(vals, seed, dist, out=out)
        ev[2 * r + 1].record()
    torch.cuda.synchronize()
    return min(ev[2 * r].elapsed_time(ev[2 * r + 1]) for r in range(reps)), out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=2000)
    ap.add_argument("--dist", default="uniform")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    rows = []
    for kind in "ABC":
        A = workloads.abnormal_paper(kind)
        cp, ri, va = (torch.from_numpy(x).to(dev) for x in (A.colptr, A.rowidx, A.vals))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        p3 = sk.Plan(cp, ri, a.d, A.m)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        p4 = sk.Plan(cp, ri, a.d, A.m, jki=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        sk.set_pair_path("kji")
        ms3, o3 = timed_apply(p3, va, a.dist, a.reps)
        sk.set_pair_path("jki")
        ms4, o4 = timed_apply(p4, va, a.dist, a.reps)
        sk.set_pair_path("auto")
        diff = float((o3 - o4).abs().max())
        st = p4.stats()
        rows.append({"pattern": f"Abnormal_{kind}", "nnz": A.nnz, "d": a.d, "dist": a.dist,
                     "alg3_plan_ms": (t1 - t0) * 1e3, "alg3_apply_ms": ms3,
                     "alg4_plan_ms": (t2 - t1) * 1e3, "alg4_apply_ms": ms4,
                     "alg4_nonzero_rows": st["jki_nonzero_rows"], "auto_builds_alg4": p3.stats()["n_items_jki"] > 0,
                     "max_abs_diff": diff})
        p3.close()
        p4.close()
    for r in rows:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
