"""Small fp4n run (development helper): random CSC, rademacher fp64, compared with the oracle.
    python scripts/f4n_small.py m n L d"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import oracle, workloads
from paper_2310_15419_b200 import sketch as sk
m, n, L, d = (int(x) for x in sys.argv[1:5])
A = workloads.random_csc(m, n, L, seed=2)
dev = torch.device("cuda:0")
plan = sk.Plan(torch.from_numpy(A.colptr).to(dev), torch.from_numpy(A.rowidx).to(dev), d, A.m, "f64")
print(plan.kernel_name("rademacher"), plan.stats())
out = plan.apply(torch.from_numpy(A.vals).to(dev), 31, "rademacher").T.cpu().numpy()
ref, B = oracle.sketch(31, "rademacher", d, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=8)
print("max err/B", float((np.abs(out - ref) / np.maximum(B, 1e-300)).max()))
