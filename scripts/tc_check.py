"""Quick GPU check of the tensor-core ±1 path against the oracle on small cases, then timing."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import workloads  # noqa: E402
from paper_2310_15419_b200 import sketch as sk  # noqa: E402


def run(A, d, seed):
    dev = torch.device("cuda:0")
    plan = sk.Plan(torch.from_numpy(A.colptr).to(dev), torch.from_numpy(A.rowidx).to(dev), d, A.m, "f64",
                   row_offset=A.row_offset)
    out = plan.apply(torch.from_numpy(A.vals).to(dev), seed, "rademacher")
    torch.cuda.synchronize()
    return out.T.cpu().numpy()


for (m, n, L, d) in [(300, 3, 5, 128), (1000, 4, 40, 300), (5000, 7, 100, 2000), (20000, 5, 3000, 700)]:
    A = workloads.random_csc(m, n, L, seed=1)
    got = run(A, d, 7)
    ref, B = oracle.sketch(7, "rademacher", d, A.m, A.n, A.colptr, A.rowidx, A.vals)
    rel = np.abs(got - ref) / np.maximum(B, 1e-300)
    print(f"m={m} n={n} L={L} d={d}: max rel err {rel.max():.3e}", flush=True)
