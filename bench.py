"""bench.py -- sketch throughput (GFLOP/s = 2·d·nnz(A)/s) of the fused on-the-fly-RNG
sketch Â = S·A on B200, 1..N GPUs (one process per GPU, torchrun), BASELINE.json metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

Default workload: config c5 (BASELINE.json configs[4]: m = 5e7, n = 1000, d = 2000, fp64,
one nonzero per row, ±1 S) -- the configuration the metric is quoted on at 1/2/4/8 GPUs.
A "step" is one sketch_apply over the whole matrix (Philox generation, transform,
multiply-accumulate, in-CTA reduction and the single store of Â: SURVEY.md §8(a) a2-a5)
plus, for N > 1, the NCCL all-reduce of the d x n partials (a6).  The plan (a1, the paper's
"format conversion") is built once and timed separately (plan_ms).
Rows of A are sharded across ranks (RNG keyed by the global row index), so the total work
is fixed as N grows ("scaling": "strong") and every rank ends with the same full Â.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402
from paper_2310_15419_b200.metrics import algorithmic_bytes, gflops  # noqa: E402


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# FP64 / FP32 vector-pipe peaks derived from unit counts and clocks (DESIGN.md §"Roofline"):
# 148 SMs x {64 fp64, 128 fp32} lanes x 2 flop per FMA x sm_max clock.
def alu_peak_tflops(dtype: str, sm_mhz: float) -> float:
    lanes = 64 if dtype == "f64" else 128
    return 148 * lanes * 2 * sm_mhz * 1e6 / 1e12


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self._t:
            self._t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def launches_per_apply(plan, dist: str, stats: dict) -> int:
    """Kernels one sketch_apply launches: the fused kernel, plus the zeroing kernel of the fp4
    path's K-split last wave when the plan made one."""
    if not (stats["n_items_rad"] or stats["n_items_pair"]):
        return 0
    split = stats.get("n_items_f4_split", 0) > 0 and "sk_rad_f4_kernel" in plan.kernel_name(dist)
    return 2 if split else 1


def load_profile_traffic(config: str, kernel: str):
    """dram bytes (read + write) per launch of `kernel` on `config` from the committed
    `ncu --set full` capture (profiles/traffic.json), or None."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            entry = json.load(f).get(config)
    except Exception:
        return None
    if isinstance(entry, dict):
        for k, v in entry.items():
            if k in kernel or kernel.startswith(k):
                return v
        return None
    return entry


def cpu_baseline(cfg, A, max_wall_s: float = 8.0):
    """The oracle, as it stands, on the host cores: a bounded sample of whole columns."""
    import oracle
    cores = oracle.max_threads()
    lens = np.diff(A.colptr)
    # grow the column sample until the run takes ~max_wall_s (bounded number of doublings)
    ncols = max(1, min(cfg.n, cores))
    best = None
    while True:
        cols = np.arange(ncols)
        As = A.select_columns(cols)
        t0 = time.perf_counter()
        oracle.sketch(cfg.seed, cfg.dist, cfg.d, As.m, As.n, As.colptr, As.rowidx, As.vals,
                      row_offset=A.row_offset, threads=cores, want_bound=False)
        dt = time.perf_counter() - t0
        best = (ncols, int(lens[:ncols].sum()), dt)
        if dt > max_wall_s / 4 or ncols >= cfg.n:
            break
        ncols = min(cfg.n, ncols * 4)
    ncols, nnz_s, dt = best
    return {"value": gflops(cfg.d, nnz_s, dt), "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
            "sample": f"{ncols} of {cfg.n} columns of {cfg.name} ({nnz_s} nnz, all d={cfg.d} rows), "
                      f"{dt:.2f} s wall"}


def run_reference(args):
    """--impl reference: the CPU oracle timed on a bounded sample of the same workload."""
    import oracle
    cfg = workloads.CONFIGS[args.config]
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    A = workloads.make_config(cfg.name) if cfg.name != "c5" else \
        workloads.make_config("c5", row_range=(0, cfg.m // 50))
    cores = oracle.max_threads()
    lens = np.diff(A.colptr)
    ncols = max(1, min(cfg.n, cores))
    # size one step to ~2-4 s of wall time
    for _ in range(6):
        As = A.select_columns(np.arange(ncols))
        t0 = time.perf_counter()
        oracle.sketch(cfg.seed, cfg.dist, cfg.d, As.m, As.n, As.colptr, As.rowidx, As.vals,
                      threads=cores, want_bound=False)
        dt = time.perf_counter() - t0
        if dt > 1.0 or ncols >= cfg.n:
            break
        ncols = min(cfg.n, ncols * 2)
    As = A.select_columns(np.arange(ncols))
    nnz_s = int(lens[:ncols].sum())
    for _ in range(args.warmup):
        oracle.sketch(cfg.seed, cfg.dist, cfg.d, As.m, As.n, As.colptr, As.rowidx, As.vals,
                      threads=cores, want_bound=False)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.sketch(cfg.seed, cfg.dist, cfg.d, As.m, As.n, As.colptr, As.rowidx, As.vals,
                      threads=cores, want_bound=False)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    v = gflops(cfg.d, nnz_s, t)
    sample = (f"{ncols} of {cfg.n} columns of {cfg.name}"
              + (" (row shard [0, m/50) of c5)" if cfg.name == "c5" else "")
              + f", {nnz_s} nnz, all d={cfg.d} rows, per step")
    print(json.dumps({
        "impl": "reference", "metric": "sketch GFLOP/s (2·d·nnz(A)/s)", "value": v,
        "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": cfg.dtype, "data": "synthetic",
        "config": {"workload": cfg.name, "m": cfg.m, "n": cfg.n, "d": cfg.d, "dist": cfg.dist,
                   "seed": cfg.seed, "sample_nnz": nnz_s},
        "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=sorted(workloads.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--shard", default="rows", choices=["rows", "cols"],
                    help="rows: row shards + NCCL all_reduce of the d x n partials (default); "
                         "cols: nnz-balanced column shards, no collective (SURVEY.md §8(f) f4)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3   # timing rule: >= 3 warm-up steps
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    import __graft_entry__
    if rank == 0:
        __graft_entry__.build()
    if world > 1:
        dist.barrier()
    from paper_2310_15419_b200 import sketch as sk

    cfg = workloads.CONFIGS[args.config]
    # ---- inputs: this rank's row shard (c5 generates shards independently) or column shard ----
    col_shard = args.shard == "cols" and world > 1
    if col_shard:
        from paper_2310_15419_b200.distributed import balanced_col_shards
        Af = workloads.make_config(cfg.name)
        cb = balanced_col_shards(Af.colptr, world)
        A = workloads.col_slice(Af, cb[rank], cb[rank + 1])
        del Af
    elif cfg.name == "c5":
        r0, r1 = workloads.shard_rows(cfg.m, world, rank)
        A = workloads.make_config("c5", row_range=(r0, r1))
    else:
        A = workloads.make_config(cfg.name)
        if world > 1:
            A = workloads.shard_csc(A, world, rank)
    nnz_local = A.nnz
    wbytes = 8 if cfg.dtype == "f64" else 4
    colptr = torch.from_numpy(A.colptr).to(dev)
    rowidx = torch.from_numpy(A.rowidx).to(dev)
    vals = torch.from_numpy(A.vals).to(dev)
    out = torch.empty((A.n, cfg.d), dtype=vals.dtype, device=dev)
    stream = torch.cuda.current_stream()
    reduce_partials = world > 1 and not col_shard

    # ---- plan (a1), timed separately: the second build (the first pays one-time driver and
    # allocator warm-up) ----
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = sk.Plan(colptr, rowidx, cfg.d, A.m, cfg.dtype, row_offset=A.row_offset)
    torch.cuda.synchronize()
    plan_first_ms = (time.perf_counter() - t0) * 1e3
    plan.close()
    t0 = time.perf_counter()
    plan = sk.Plan(colptr, rowidx, cfg.d, A.m, cfg.dtype, row_offset=A.row_offset)
    torch.cuda.synchronize()
    plan_ms = (time.perf_counter() - t0) * 1e3

    # L2 policy: inputs larger than the 126 MB L2 need no flush; smaller ones get a flush.
    in_bytes = algorithmic_bytes(cfg.d, cfg.n, nnz_local, wbytes)
    flush = None
    if in_bytes < 256 * 2**20:
        flush = torch.empty(512 * 2**20 // 4, dtype=torch.int32, device=dev)

    def step():
        plan.apply(vals, cfg.seed, cfg.dist, out=out)
        if reduce_partials:
            dist.all_reduce(out, op=dist.ReduceOp.SUM)

    for _ in range(args.warmup):
        if flush is not None:
            flush.zero_()
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    mids = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        if flush is not None:
            flush.zero_()
        starts[i].record(stream)
        plan.apply(vals, cfg.seed, cfg.dist, out=out)
        mids[i].record(stream)
        if reduce_partials:
            dist.all_reduce(out, op=dist.ReduceOp.SUM)
        ends[i].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    kern_ms = [s.elapsed_time(m) for s, m in zip(starts, mids)]
    t_step = sum(step_ms) / len(step_ms)
    t_kern = sum(kern_ms) / len(kern_ms)
    if world > 1:
        tt = torch.tensor([t_step, t_kern], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, t_kern = float(tt[0]), float(tt[1])
    if world > 1:
        nn = torch.tensor([nnz_local], dtype=torch.int64, device=dev)
        dist.all_reduce(nn)
        nnz_total = int(nn.item())
    else:
        nnz_total = nnz_local
    value = gflops(cfg.d, nnz_total, t_step / 1e3)

    # ---- e2e through the host-buffer C-ABI entry point (pinned buffers) ----
    e2e = None
    if not args.no_e2e:
        h_colptr = torch.from_numpy(A.colptr).pin_memory()
        h_rowidx = torch.from_numpy(A.rowidx).pin_memory()
        h_vals = torch.from_numpy(A.vals).pin_memory()
        h_out = torch.empty((A.n, cfg.d), dtype=vals.dtype).pin_memory()
        for _ in range(2):
            sk.sketch_apply_host(cfg.seed, cfg.dist, cfg.d, A.m, h_colptr, h_rowidx, h_vals,
                                 out=h_out, row_offset=A.row_offset)
        if world > 1:
            dist.barrier()
        e_times = []
        for _ in range(max(3, min(args.steps, 5))):
            t0 = time.perf_counter()
            sk.sketch_apply_host(cfg.seed, cfg.dist, cfg.d, A.m, h_colptr, h_rowidx, h_vals,
                                 out=h_out, row_offset=A.row_offset)
            e_times.append(time.perf_counter() - t0)
        te = sum(e_times) / len(e_times)
        if world > 1:
            tt = torch.tensor([te], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt[0])
        h2d = A.colptr.nbytes + A.rowidx.nbytes + A.vals.nbytes
        e2e = {"value": gflops(cfg.d, nnz_total, te), "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(A.n * cfg.d * wbytes),
               "ms_per_step": te * 1e3,
               "note": "sketch_apply_host: pinned host A -> device, plan, fused apply, Â -> host; "
                       "column groups pipelined on copy streams" + ("; no cross-GPU reduce" if world > 1 else "")}

    # ---- roofline of the dominant kernel (the fused apply; one launch per step) ----
    peaks, peak_src = _peaks()
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    achieved_tf = 2.0 * cfg.d * nnz_local / (t_kern / 1e3) / 1e12
    peak_tf = alu_peak_tflops(cfg.dtype, sm_mhz)
    stats = plan.stats()
    kname = plan.kernel_name(cfg.dist)
    roofline = {"bound": "alu", "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
                "frac": achieved_tf / peak_tf, "traffic": load_profile_traffic(cfg.name, kname),
                "kernel": kname,
                "peak_source": f"{cfg.dtype} vector pipe (the SpMM's FMA roofline): 148 SMs x "
                               f"{64 if cfg.dtype == 'f64' else 128} lanes x 2 flop x {sm_mhz:.0f} MHz "
                               f"(sm_max_mhz of {peak_src} peaks)",
                "kernel_ms": t_kern,
                "hbm_frac": (in_bytes / (t_kern / 1e3) / 1e9) / float(peaks.get("hbm_gbs", 6650.0)),
                "algorithmic_bytes": int(in_bytes)}
    if "mxf4" in kname:
        # the tensor-core path's own ceiling: one M=128,K=64 mxf4 MMA per 92 cycles
        # (scripts/microbench_mxf4.cu) = 89 (row, nonzero) entries/clk/SM
        tc_peak = 2 * 89.0 * 148 * sm_mhz * 1e6 / 1e12
        roofline["tensor_feed_peak"] = tc_peak
        roofline["tensor_feed_frac"] = achieved_tf / tc_peak

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, A)

    if rank == 0:
        line = {
            "metric": "sketch GFLOP/s (2·d·nnz(A)/s)", "value": value, "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": cfg.dtype, "data": "synthetic",
            "config": {"workload": cfg.name, "m": cfg.m, "n": cfg.n, "d": cfg.d, "dist": cfg.dist,
                       "seed": cfg.seed, "nnz": nnz_total,
                       "parallelism": f"{'cols' if col_shard else 'rows'}{world}",
                       "l2": "inputs > L2 (no flush)" if flush is None else "L2 flushed between steps",
                       "plan_ms": plan_ms, "plan_first_ms": plan_first_ms, "kernel_ms": t_kern,
                       "reduce": "NCCL all_reduce of d x n partials" if reduce_partials else None},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clocks, "gpu_launches": args.steps * launches_per_apply(plan, cfg.dist, stats),
        }
        print(json.dumps(line))
    plan.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
