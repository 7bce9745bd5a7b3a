"""Algorithm 3 (kji) vs forced Algorithm 4 (jki) across row reuse: n = 1000 columns of 1000 nonzeros
drawn from R rows (R from 4e6 down to 3000), d = 2000, uniform and Gaussian, f64 and f32.  Prints one
JSON line per (R, dtype, dist) with the measured reuse nnz / jki_rows and both apply times (median
of 5 after 2 warm-ups, L2 flushed) -- the data behind the plan's automatic choice.

    python scripts/jki_reuse_sweep.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2310_15419_b200 import sketch as sk  # noqa: E402
from jki_configs import med_ms  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    d = 2000
    for R in (4_000_000, 1_000_000, 300_000, 100_000, 30_000, 10_000, 3_000):
        A = workloads.random_csc(R, 1000, 1000, seed=R % 1000 + 7)
        for dt in ("f64", "f32"):
            vals = A.vals.astype(np.float32 if dt == "f32" else np.float64)
            cp, ri, va = (torch.from_numpy(x).to(dev) for x in (A.colptr, A.rowidx, vals))
            out = torch.empty((A.n, d), dtype=va.dtype, device=dev)
            p3 = sk.Plan(cp, ri, d, A.m, dt)
            p4 = sk.Plan(cp, ri, d, A.m, dt, jki=True)
            st = p4.stats()
            auto = p3.stats()["n_items_jki"] > 0
            for dist in ("uniform", "gaussian"):
                sk.set_pair_path("kji")
                ms3 = med_ms(p3, va, dist, out, flush)
                sk.set_pair_path("jki")
                ms4 = med_ms(p4, va, dist, out, flush)
                sk.set_pair_path("auto")
                print(json.dumps({"R": R, "dtype": dt, "dist": dist, "nnz": A.nnz, "jki_rows": st["jki_nonzero_rows"],
                                  "reuse": round(A.nnz / max(st["jki_nonzero_rows"], 1), 3), "kji_ms": round(ms3, 4),
                                  "jki_ms": round(ms4, 4), "auto_built": auto,
                                  "auto_kernel": p3.kernel_name(dist)}), flush=True)
            p3.close()
            p4.close()


if __name__ == "__main__":
    main()
