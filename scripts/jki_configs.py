"""Algorithm 3 (kji) vs a forced Algorithm 4 (jki, b_n = jki_block_cols) on BASELINE configs c2 / c3
with both distributions: apply ms (median of 5 after 2 warm-ups, L2 flushed), plan ms, reuse.

    python scripts/jki_configs.py [c2 c3 ...]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2310_15419_b200 import sketch as sk  # noqa: E402


def med_ms(plan, vals, dist, out, flush, reps=5, warm=2):
    ts = []
    for r in range(warm + reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.apply(vals, 7, dist, out=out)
        b.record()
        torch.cuda.synchronize()
        if r >= warm:
            ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    names = sys.argv[1:] or ["c2", "c3"]
    dev = torch.device("cuda:0")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for name in names:
        cfg = workloads.CONFIGS[name]
        A = workloads.make_config(name)
        cp, ri, va = (torch.from_numpy(x).to(dev) for x in (A.colptr, A.rowidx, A.vals))
        out = torch.empty((A.n, cfg.d), dtype=va.dtype, device=dev)
        dt = "f64" if A.vals.dtype == np.float64 else "f32"
        p3 = sk.Plan(cp, ri, cfg.d, A.m, dt)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        p4 = sk.Plan(cp, ri, cfg.d, A.m, dt, jki=True)
        torch.cuda.synchronize()
        plan_ms = (time.perf_counter() - t0) * 1e3
        st = p4.stats()
        for dist in ("uniform", "gaussian"):
            sk.set_pair_path("kji")
            ms3 = med_ms(p3, va, dist, out, flush)
            o3 = out.clone()
            sk.set_pair_path("jki")
            ms4 = med_ms(p4, va, dist, out, flush)
            sk.set_pair_path("auto")
            diff = float((o3 - out).abs().max() / max(float(o3.abs().max()), 1e-300))
            print(json.dumps({"config": name, "dist": dist, "d": cfg.d, "nnz": A.nnz,
                              "jki_rows": st["jki_nonzero_rows"], "reuse": A.nnz / max(st["jki_nonzero_rows"], 1),
                              "kji_ms": ms3, "jki_ms": ms4, "jki_plan_ms": plan_ms, "rel_diff": diff,
                              "n_items_jki": st["n_items_jki"]}), flush=True)
        p3.close()
        p4.close()


if __name__ == "__main__":
    main()
