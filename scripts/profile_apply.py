"""Minimal driver for ncu: build config A, plan once, run sketch_apply `--reps` times.

    python scripts/profile_apply.py --config c5 --reps 3
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2310_15419_b200 import sketch as sk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--rows", type=int, default=0, help="c5 only: use rows [0, rows)")
    ap.add_argument("--dist", default=None, help="override the config's distribution")
    ap.add_argument("--f32", action="store_true", help="values rounded to fp32 (fp32 arithmetic)")
    ap.add_argument("--jki", action="store_true", help="forced Algorithm 4 plan and path")
    a = ap.parse_args()
    cfg = workloads.CONFIGS[a.config]
    A = workloads.make_config(cfg.name, row_range=(0, a.rows)) if a.rows else workloads.make_config(cfg.name)
    dist = a.dist or cfg.dist
    dtype = "f32" if a.f32 else cfg.dtype
    if a.f32:
        A.vals = A.vals.astype("float32")
    dev = torch.device("cuda:0")
    colptr = torch.from_numpy(A.colptr).to(dev)
    rowidx = torch.from_numpy(A.rowidx).to(dev)
    vals = torch.from_numpy(A.vals).to(dev)
    plan = sk.Plan(colptr, rowidx, cfg.d, A.m, dtype, row_offset=A.row_offset, jki=a.jki)
    if a.jki:
        sk.set_pair_path("jki")
    out = torch.empty((cfg.n, cfg.d), dtype=vals.dtype, device=dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * a.reps)]
    for r in range(a.reps):
        ev[2 * r].record()
        plan.apply(vals, cfg.seed, dist, out=out)
        ev[2 * r + 1].record()
    torch.cuda.synchronize()
    print(a.config, dist, dtype, plan.kernel_name(dist), "nnz", A.nnz, "stats", plan.stats())
    print("ms", [round(ev[2 * r].elapsed_time(ev[2 * r + 1]), 3) for r in range(a.reps)])
    plan.close()


if __name__ == "__main__":
    main()
