"""Quick GPU check of every ±1 fp64 kernel path against the oracle on small cases."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import workloads  # noqa: E402
from paper_2310_15419_b200 import sketch as sk  # noqa: E402

paths = sys.argv[1:] or ["fp4", "hybrid", "int8smem", "int8tmem", "simt"]
dev = torch.device("cuda:0")
for path in paths:
    sk.set_rad_f64_path(path)
    worst = 0.0
    for (m, n, L, d) in [(3000, 3, 500, 128), (10000, 4, 400, 300), (50000, 7, 1000, 2000), (20000, 5, 3000, 700),
                         (90000, 300, 260, 2000)]:
        A = workloads.random_csc(m, n, L, seed=1)
        plan = sk.Plan(torch.from_numpy(A.colptr).to(dev), torch.from_numpy(A.rowidx).to(dev), d, A.m, "f64")
        out = plan.apply(torch.from_numpy(A.vals).to(dev), 7, "rademacher")
        torch.cuda.synchronize()
        got = out.T.cpu().numpy()
        kname = plan.kernel_name("rademacher")
        plan.close()
        ref, B = oracle.sketch(7, "rademacher", d, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=8)
        worst = max(worst, float((np.abs(got - ref) / np.maximum(B, 1e-300)).max()))
    print(f"{path:9s} {kname}: max rel err {worst:.3e}", flush=True)
