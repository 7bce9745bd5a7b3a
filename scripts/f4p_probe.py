"""Small persistent-f4 probe: n columns of L nonzeros, d rows, compared with the oracle."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import oracle, workloads
from paper_2310_15419_b200 import sketch as sk
n, L, d = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
A = workloads.random_csc(200000, n, L, seed=5)
dev = torch.device("cuda:0")
t = lambda x: torch.from_numpy(x).to(dev)
plan = sk.Plan(t(A.colptr), t(A.rowidx), d, A.m)
print(plan.kernel_name("rademacher"), plan.stats()["n_items_f4"], flush=True)
out = plan.apply(t(A.vals), 3, "rademacher").T.cpu().numpy()
ref, B = oracle.sketch(3, "rademacher", d, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=8)
err = np.abs(out - ref) / np.maximum(B, 1e-300)
print("max err/B", float(err.max()), "ok", bool(np.all(np.abs(out - ref) <= 1e-12 * B)))
