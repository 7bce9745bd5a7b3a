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
`--gpus N` without torchrun's environment starts the N ranks itself (torch.distributed.run on
127.0.0.1).  At N = 1 the line also carries `per_config`: c1-c4 timed in the same process with
their strict roofline fractions (G = ceil(d/E) nnzrows, paper_2310_15419_b200/
metrics.py roofline()).
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
    """Kernels of the library one sketch_apply launches.  ±1: the tensor-core kernel with its IEEE fix-up
    of non-finite columns (and the zeroing of the K-split rows when the plan split its last wave) when columns of 896 ..
    131071 nonzeros exist (fp64), the SIMT kernel for the other columns, and for fp32 the IEEE fix-up
    scan.  Uniform / Gaussian: the fused kernel, or Algorithm 4's gather + kernel (+ the finishing sum
    of split column blocks)."""
    if dist == "rademacher":
        f4 = int(stats.get("n_items_f4", 0) > 0)
        n = 2 * f4 + int(f4 and stats.get("n_items_f4_split", 0) > 0) + int(stats["n_items_rad"] > 0)
        if "sk_rad_kernel<float>" in plan.kernel_name(dist) and stats["n_items_rad"] > 0:
            n += 1
        return n
    if stats.get("n_items_jki", 0) > 0 and "Algorithm 4" in plan.kernel_name(dist):
        return 3
    return int(stats["n_items_pair"] > 0)


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
    """The oracle, as it stands, on the host cores: a bounded sample of whole columns.  (Under torchrun
    OMP_NUM_THREADS is 1; rank 0 runs this after the timed region while the other ranks wait, so it
    takes every core of the host.)"""
    import oracle
    cores = max(oracle.max_threads(), os.cpu_count() or 1)
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


def _free_port() -> int:
    import socket
    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        return sck.getsockname()[1]


def relaunch_under_torchrun(n: int) -> int:
    """`bench.py --gpus N` without a torchrun environment: start the N ranks ourselves (one process
    per GPU, rendezvous on 127.0.0.1) with the same arguments; rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def nonzero_rows(A) -> int:
    """nnzrows(A): rows holding at least one stored entry (the strict RNG count's row factor)."""
    if A.nnz == 0:
        return 0
    return int(np.count_nonzero(np.bincount(A.rowidx, minlength=A.m)))


def time_applies(torch, plan, vals, seed, dist_name, out, steps, warmup, flush, stream, after=None):
    """Per-step device times (CUDA events on the launching stream) of plan.apply (+ `after`, e.g. the
    cross-GPU reduce): returns (apply ms list, step ms list)."""
    for _ in range(warmup):
        if flush is not None:
            flush.zero_()
        plan.apply(vals, seed, dist_name, out=out)
        if after:
            after()
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    for i in range(steps):
        if flush is not None:
            flush.zero_()
        ev[i][0].record(stream)
        plan.apply(vals, seed, dist_name, out=out)
        ev[i][1].record(stream)
        if after:
            after()
        ev[i][2].record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b, _ in ev], [a.elapsed_time(c) for a, _, c in ev]


def per_config_lines(torch, sk, dev, names, steps, warmup, peaks, sm_mhz):
    """The other BASELINE.json configs, each timed in this process (N = 1): apply ms (median of
    `steps` after `warmup`, L2 flushed between steps when the inputs fit in L2), GFLOP/s and the
    strict roofline fraction of SURVEY.md §8(d)."""
    from paper_2310_15419_b200.metrics import roofline, roofline_report
    res = {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    for name in names:
        cfg = workloads.CONFIGS[name]
        A = workloads.make_config(name)
        colptr = torch.from_numpy(A.colptr).to(dev)
        rowidx = torch.from_numpy(A.rowidx).to(dev)
        vals = torch.from_numpy(A.vals).to(dev)
        out = torch.empty((A.n, cfg.d), dtype=vals.dtype, device=dev)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan = sk.Plan(colptr, rowidx, cfg.d, A.m, cfg.dtype)
        torch.cuda.synchronize()
        plan_ms = (time.perf_counter() - t0) * 1e3
        w = 8 if cfg.dtype == "f64" else 4
        flush = torch.empty(512 * 2**20 // 4, dtype=torch.int32, device=dev) \
            if algorithmic_bytes(cfg.d, cfg.n, A.nnz, w) < 256 * 2**20 else None
        k_ms, _ = time_applies(torch, plan, vals, cfg.seed, cfg.dist, out, steps, warmup, flush,
                               torch.cuda.current_stream())
        t = statistics.median(k_ms)
        nzr = nonzero_rows(A)
        rl = roofline(cfg.dist, cfg.dtype, cfg.d, cfg.n, A.nnz, nzr, hbm, sm_mhz)
        rep = roofline_report(rl, t / 1e3, cfg.dtype, hbm, sm_mhz)
        st = plan.stats()
        res[name] = {"ms": t, "ms_min": min(k_ms), "gflops": gflops(cfg.d, A.nnz, t / 1e3),
                     "bound": rep["bound"], "frac": rep["frac"], "t_roof_ms": rep["t_roof_ms"],
                     "achieved": rep["achieved"], "peak": rep["peak"], "unit": rep["unit"],
                     "kernel": plan.kernel_name(cfg.dist), "dist": cfg.dist, "dtype": cfg.dtype,
                     "traffic": load_profile_traffic(name, plan.kernel_name(cfg.dist)),
                     "d": cfg.d, "n": cfg.n, "m": cfg.m, "nnz": A.nnz, "nnzrows": nzr,
                     "g_calls_strict": rl["g_calls_strict"], "g_calls_alg3": rl["g_calls_alg3"],
                     "plan_ms": plan_ms, "launches_per_step": launches_per_apply(plan, cfg.dist, st),
                     "l2": "L2 flushed between steps" if flush is not None else "inputs > L2 (no flush)"}
        plan.close()
        del flush, colptr, rowidx, vals, out
        torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=sorted(workloads.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--shard", default="rows", choices=["rows", "cols"],
                    help="rows: row shards + all_reduce of the d x n partials (default); "
                         "cols: nnz-balanced column shards, no collective (SURVEY.md §8(f) f4)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3   # timing rule: >= 3 warm-up steps
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args.gpus)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    ndev = torch.cuda.device_count()
    if ndev == 0:
        raise SystemExit("bench.py needs a CUDA device (there is no CPU fallback)")
    # One process per GPU over NCCL.  With fewer GPUs than ranks (a functional run on a small box)
    # the ranks share devices and the partials are summed through gloo (host-staged): such a line
    # says "shared_gpus": true and is not a scaling measurement.
    shared = world > ndev
    torch.cuda.set_device(local % ndev)
    dev = torch.device("cuda", local % ndev)
    backend = "gloo" if shared else "nccl"
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    import __graft_entry__
    if rank == 0:
        __graft_entry__.build()
    if world > 1:
        dist.barrier()
    from paper_2310_15419_b200 import sketch as sk
    from paper_2310_15419_b200 import distributed as skd
    from paper_2310_15419_b200.metrics import roofline, roofline_report

    cfg = workloads.CONFIGS[args.config]
    # ---- inputs: this rank's row shard (c5 generates shards independently) or column shard ----
    col_shard = args.shard == "cols" and world > 1
    if col_shard:
        Af = workloads.make_config(cfg.name)
        cb = skd.balanced_col_shards(Af.colptr, world)
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
    in_bytes = algorithmic_bytes(cfg.d, A.n, nnz_local, wbytes)
    flush = None
    if in_bytes < 256 * 2**20:
        flush = torch.empty(512 * 2**20 // 4, dtype=torch.int32, device=dev)

    def do_reduce():
        skd.reduce_partials(out, mode="all_reduce")
        if shared:
            torch.cuda.synchronize()     # gloo: host-staged; keep the events honest

    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local % ndev)
    sampler.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    kern_ms, step_ms = time_applies(torch, plan, vals, cfg.seed, cfg.dist, out, args.steps, args.warmup, flush,
                                    stream, do_reduce if reduce_partials else None)
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    t_step = sum(step_ms) / len(step_ms)
    t_kern = sum(kern_ms) / len(kern_ms)
    t_red = t_step - t_kern
    if world > 1:
        tt = torch.tensor([t_step, t_kern, t_red], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, t_kern, t_red = float(tt[0]), float(tt[1]), float(tt[2])
        nn = torch.tensor([nnz_local], dtype=torch.int64, device=dev)
        dist.all_reduce(nn)
        nnz_total = int(nn.item())
    else:
        nnz_total = nnz_local
    value = gflops(cfg.d, nnz_total, t_step / 1e3)

    # ---- e2e through the host-buffer C-ABI entry point (pinned buffers; + the reduce at N > 1) ----
    e2e = None
    if not args.no_e2e:
        h_colptr = torch.from_numpy(A.colptr).pin_memory()
        h_rowidx = torch.from_numpy(A.rowidx).pin_memory()
        h_vals = torch.from_numpy(A.vals).pin_memory()
        h_out = torch.empty((A.n, cfg.d), dtype=vals.dtype).pin_memory()

        def e2e_step():
            if reduce_partials:
                skd.sketch_row_sharded_e2e(h_colptr, h_rowidx, h_vals, cfg.d, A.m, A.row_offset, cfg.seed,
                                           cfg.dist, h_out, work=out)
            else:
                sk.sketch_apply_host(cfg.seed, cfg.dist, cfg.d, A.m, h_colptr, h_rowidx, h_vals,
                                     out=h_out, row_offset=A.row_offset)
        for _ in range(2):
            e2e_step()
        e_times = []
        for _ in range(max(3, min(args.steps, 5))):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            e2e_step()
            e_times.append(time.perf_counter() - t0)
        te = sum(e_times) / len(e_times)
        h2d = A.colptr.nbytes + A.rowidx.nbytes + A.vals.nbytes
        d2h = A.n * cfg.d * wbytes
        if world > 1:
            tt = torch.tensor([te], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt[0])
            bb = torch.tensor([h2d, d2h], dtype=torch.int64, device=dev)
            dist.all_reduce(bb)
            h2d, d2h = int(bb[0]), int(bb[1])
        e2e = {"value": gflops(cfg.d, nnz_total, te), "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": te * 1e3,
               "note": "sketch_apply_host: pinned host A -> device, plan, fused apply, Â -> host; column groups "
                       "pipelined on copy streams" +
                       ("; per rank into device memory, then the all_reduce of the partials and Â -> pinned host "
                        "(bytes summed over ranks; wall clock, max over ranks)" if reduce_partials else "")}

    # ---- roofline of the dominant kernel on this rank (strict G = ceil(d/E) nnzrows) ----
    peaks, peak_src = _peaks()
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    stats = plan.stats()
    kname = plan.kernel_name(cfg.dist)
    nzr = nonzero_rows(A)
    rl = roofline(cfg.dist, cfg.dtype, cfg.d, A.n, nnz_local, nzr, hbm, sm_mhz)
    rep = roofline_report(rl, t_kern / 1e3, cfg.dtype, hbm, sm_mhz)
    roof = {"bound": rep["bound"], "achieved": rep["achieved"], "peak": rep["peak"], "unit": rep["unit"],
            "frac": rep["frac"], "traffic": load_profile_traffic(cfg.name, kname), "kernel": kname,
            "kernel_ms": t_kern, "t_roof_ms": rep["t_roof_ms"],
            "peak_source": {"fp64_pipe": f"148 SMs x 64 FP64 lanes x 2 flop x {sm_mhz:.0f} MHz (sm_max_mhz of "
                                         f"{peak_src} peaks)",
                            "fp32_pipe": f"148 SMs x 128 FP32 lanes x 2 flop x {sm_mhz:.0f} MHz (sm_max_mhz of "
                                         f"{peak_src} peaks)",
                            "int_philox": "Philox4x32-10 blocks/s measured on B200 (profiles/r01_microbench.json)",
                            "hbm": f"hbm_gbs of {peak_src} peaks"}[rep["bound"]],
            "model": {"t_hbm_ms": rl["t_hbm"] * 1e3, "t_fp_ms": rl["t_fp"] * 1e3, "t_int_ms": rl["t_int"] * 1e3,
                      "nnzrows": nzr, "g_calls_strict": rl["g_calls_strict"], "g_calls_alg3": rl["g_calls_alg3"],
                      "algorithmic_bytes": rl["algorithmic_bytes"]},
            "hbm_frac": (rl["algorithmic_bytes"] / (t_kern / 1e3) / 1e9) / hbm,
            "scope": "rank 0's kernel on its shard" if world > 1 else "the whole matrix"}
    if "mxf4" in kname:
        # the tensor-core path's own ceiling: one M=128,K=64 mxf4 MMA per 92 cycles with the A tile
        # streamed from shared memory (scripts/microbench_mxf4.cu) = 89 (row, nonzero) entries/clk/SM
        tc_peak = 2 * 89.0 * 148 * sm_mhz * 1e6 / 1e12
        roof["tensor_feed_peak"] = tc_peak
        roof["tensor_feed_frac"] = 2.0 * cfg.d * nnz_local / (t_kern / 1e3) / 1e12 / tc_peak

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, A)
        if world > 1:
            cpu["sample"] += f" (rank 0's row shard of {world})"
    per_config = None
    if rank == 0 and world == 1 and not args.no_per_config:
        others = [c for c in ("c1", "c2", "c3", "c4", "c5") if c != cfg.name]
        per_config = per_config_lines(torch, sk, dev, others, max(5, args.steps), args.warmup, peaks, sm_mhz)
        per_config[cfg.name] = {"ms": t_kern, "gflops": gflops(cfg.d, nnz_local, t_kern / 1e3),
                                "bound": rep["bound"], "frac": rep["frac"], "t_roof_ms": rep["t_roof_ms"],
                                "kernel": kname, "nnz": nnz_local, "nnzrows": nzr, "note": "the headline run above"}
    if world > 1:
        dist.barrier()

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
                       "reduce": ({"op": "all_reduce (sum of the d x n partials)", "backend": backend,
                                   "bytes": A.n * cfg.d * wbytes, "ms": t_red,
                                   "bus_gbs": 2 * (world - 1) / world * A.n * cfg.d * wbytes / (t_red / 1e3) / 1e9
                                   if t_red > 0 else None} if reduce_partials else None),
                       "shared_gpus": shared},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "per_config": per_config,
            "clocks": clocks, "gpu_launches": args.steps * launches_per_apply(plan, cfg.dist, stats),
        }
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
