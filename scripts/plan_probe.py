"""Plan-time breakdown (SKETCH_TIMING=1 prints the phases) for a config.

    SKETCH_TIMING=1 python scripts/plan_probe.py --config c5
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2310_15419_b200 import sketch as sk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    a = ap.parse_args()
    cfg = workloads.CONFIGS[a.config]
    A = workloads.make_config(cfg.name)
    colptr = torch.from_numpy(A.colptr).cuda()
    rowidx = torch.from_numpy(A.rowidx).cuda()
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan = sk.Plan(colptr, rowidx, cfg.d, A.m, cfg.dtype)
        t = time.perf_counter() - t0
        plan.close()
        print(f"{a.config} plan {t * 1e3:.2f} ms", flush=True)


if __name__ == "__main__":
    main()
