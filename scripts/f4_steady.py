"""Steady-state per-stage cost of the two tensor-core kernels: n columns of L nonzeros, d rows (one
item per column when d <= 768), timed per-item vs persistent (CUDA events, median of 7)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import workloads
from paper_2310_15419_b200 import sketch as sk
n, L, d = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
A = workloads.random_csc(1_000_000, n, L, seed=5)
dev = torch.device("cuda:0")
t = lambda x: torch.from_numpy(x).to(dev)
cp, ri, va = t(A.colptr), t(A.rowidx), t(A.vals)
for mode in ("off", "on", "off", "on"):
    sk.set_f4_persistent(mode)
    plan = sk.Plan(cp, ri, d, A.m)
    out = torch.empty((n, d), dtype=torch.float64, device=dev)
    ts = []
    for r in range(9):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); plan.apply(va, 3, "rademacher", out=out); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    st = plan.stats()
    print(mode, plan.kernel_name("rademacher")[:18], "items", st["n_items_f4"], "ms", round(float(np.median(ts[2:])), 4), flush=True)
    plan.close()
