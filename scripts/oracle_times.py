"""The CPU oracle timed on every BASELINE.json config on this host's cores: whole
matrix for c1-c4, and c5 in full (about a minute on 16 cores).  Prints one JSON line per config.

    python scripts/oracle_times.py [--configs c1,c2,...]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import workloads  # noqa: E402
from paper_2310_15419_b200.metrics import gflops  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    a = ap.parse_args()
    oracle.build()
    cores = oracle.max_threads()
    model = ""
    try:
        model = [ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo") if ln.startswith("model name")][0]
    except Exception:
        pass
    for name in a.configs.split(","):
        cfg = workloads.CONFIGS[name]
        A = workloads.make_config(name)
        nzr = int(np.count_nonzero(np.bincount(A.rowidx, minlength=A.m)))
        t0 = time.perf_counter()
        oracle.sketch(cfg.seed, cfg.dist, cfg.d, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=cores, want_bound=False)
        dt = time.perf_counter() - t0
        print(json.dumps({"config": name, "cores": cores, "cpu": model, "seconds": dt, "gflops": gflops(cfg.d, A.nnz, dt),
                          "nnz": A.nnz, "nnzrows": nzr, "d": cfg.d, "n": cfg.n, "m": cfg.m, "dist": cfg.dist,
                          "dtype": cfg.dtype}), flush=True)


if __name__ == "__main__":
    main()
