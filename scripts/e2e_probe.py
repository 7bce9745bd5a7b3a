"""End-to-end (host buffers) breakdown on c5: pinned H2D bandwidth alone, and sketch_apply_host
wall time for several column-group counts.

    python scripts/e2e_probe.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2310_15419_b200 import sketch as sk  # noqa: E402


def main():
    cfg = workloads.CONFIGS["c5"]
    A = workloads.make_config("c5")
    h_colptr = torch.from_numpy(A.colptr).pin_memory()
    h_rowidx = torch.from_numpy(A.rowidx).pin_memory()
    h_vals = torch.from_numpy(A.vals).pin_memory()
    h_out = torch.empty((A.n, cfg.d), dtype=h_vals.dtype).pin_memory()
    d_rowidx = torch.empty_like(h_rowidx, device="cuda")
    d_vals = torch.empty_like(h_vals, device="cuda")
    for _ in range(3):
        t0 = time.perf_counter()
        d_rowidx.copy_(h_rowidx, non_blocking=True)
        d_vals.copy_(h_vals, non_blocking=True)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
    nbytes = h_rowidx.numel() * 4 + h_vals.numel() * 8
    print(f"H2D {nbytes / 1e6:.0f} MB: {t * 1e3:.2f} ms = {nbytes / t / 1e9:.1f} GB/s")
    d_out = torch.empty((A.n, cfg.d), dtype=h_vals.dtype, device="cuda")
    for _ in range(3):
        t0 = time.perf_counter()
        h_out.copy_(d_out, non_blocking=True)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
    print(f"D2H {d_out.numel() * 8 / 1e6:.0f} MB: {t * 1e3:.2f} ms")
    for G in (0, 2, 4, 8, 16, 32):
        ts = []
        for _ in range(4):
            t0 = time.perf_counter()
            sk.sketch_apply_host(cfg.seed, cfg.dist, cfg.d, A.m, h_colptr, h_rowidx, h_vals, out=h_out,
                                 pipeline_chunks=G)
            ts.append(time.perf_counter() - t0)
        print(f"apply_host groups={G}: " + " ".join(f"{x * 1e3:.2f}" for x in ts) + " ms")
    t0 = time.perf_counter()
    plan = sk.Plan(d_rowidx.new_tensor(A.colptr, dtype=torch.int64) if False else torch.from_numpy(A.colptr).cuda(),
                   d_rowidx, cfg.d, A.m, "f64")
    torch.cuda.synchronize()
    print(f"device plan: {(time.perf_counter() - t0) * 1e3:.2f} ms")
    plan.close()


if __name__ == "__main__":
    main()
