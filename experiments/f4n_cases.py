"""Run the fp4n edge cases of tests/test_gpu_parity.py one by one (development helper)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import oracle, workloads
from paper_2310_15419_b200 import sketch as sk
i = int(sys.argv[1])
cases = [lambda: workloads.random_csc(50000, 40, 300, seed=2),
         lambda: workloads.random_csc(30000, 12, [0, 500, 0, 0, 640, 1, 0, 3300, 0, 2, 0, 100], seed=5),
         lambda: workloads.random_csc(200000, 24, [20000] + [10] * 23, seed=6),
         lambda: workloads.random_csc(5000, 10, 400, seed=7, sorted_rows=False, duplicates=True),
         lambda: workloads.random_csc(40000, 6, 700, seed=17)]
ds = [1000, 300, 1100, 129, 2050]
A, d = cases[i](), ds[i]
dev = torch.device("cuda:0")
plan = sk.Plan(torch.from_numpy(A.colptr).to(dev), torch.from_numpy(A.rowidx).to(dev), d, A.m, "f64")
if os.environ.get("SKETCH_RAD_F64_PATH"): sk.set_rad_f64_path(os.environ["SKETCH_RAD_F64_PATH"])
print(i, plan.kernel_name("rademacher"), plan.stats(), flush=True)
out = plan.apply(torch.from_numpy(A.vals).to(dev), 31, "rademacher").T.cpu().numpy()
ref, B = oracle.sketch(31, "rademacher", d, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=8)
print("max err/B", float((np.abs(out - ref) / np.maximum(B, 1e-300)).max()))
