"""Minimal driver for ncu of the Algorithm 4 kernel: Abnormal_A (PAPER.md:679-707 pattern), d = 2000,
forced jki plan, `--reps` applies of `--dist`."""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import workloads  # noqa: E402
from paper_2310_15419_b200 import sketch as sk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dist", default="gaussian")
ap.add_argument("--kind", default="A")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
A = workloads.abnormal_paper(a.kind)
dev = torch.device("cuda:0")
cp, ri, va = (torch.from_numpy(x).to(dev) for x in (A.colptr, A.rowidx, A.vals))
plan = sk.Plan(cp, ri, 2000, A.m, jki=True)
sk.set_pair_path("jki")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * a.reps)]
for r in range(a.reps):
    ev[2 * r].record()
    plan.apply(va, 5, a.dist)
    ev[2 * r + 1].record()
torch.cuda.synchronize()
print(plan.kernel_name(a.dist), plan.stats()["jki_nonzero_rows"], "ms", [round(ev[2 * r].elapsed_time(ev[2 * r + 1]), 3) for r in range(a.reps)])
