"""Host-side pieces of bench.py's JSON line (no GPU): peaks, launch counting, traffic lookup,
and the metric / byte arithmetic it reports."""
import json
import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2310_15419_b200.metrics import algorithmic_bytes, gflops  # noqa: E402


def test_strict_roofline_matches_survey_model():
    # SURVEY.md §8(d) d.3 / VERDICT r1: c2 is Philox-bound at ceil(d/2) nnzrows blocks (1.39 ms at the
    # measured 4.549e11 blocks/s), c3 (reading A: 871,836 nnz, 783,968 nonzero rows) Philox-bound at
    # 5.17 ms with the FP64 term at 5.08 ms (38 FP64 ops per pair), c4 FP32-bound at 0.537 ms, c5
    # FP64-bound at 5.37 ms -- all at 1965 MHz and 6544 GB/s
    from paper_2310_15419_b200.metrics import roofline, roofline_report
    c2 = roofline("uniform", "f64", 2000, 1000, 1_000_000, 632_695, 6544, 1965)
    assert c2["bound"] == "int_philox" and c2["t_roof"] * 1e3 == pytest.approx(1.3908, rel=1e-3)
    assert c2["g_calls_strict"] == 1000 * 632_695 and c2["g_calls_alg3"] == 1000 * 1_000_000
    assert roofline_report(c2, 2.71e-3, "f64", 6544, 1965)["frac"] == pytest.approx(0.513, abs=2e-3)
    c3 = roofline("gaussian", "f64", 6000, 2000, 871_836, 783_968, 6544, 1965)
    assert c3["bound"] == "int_philox" and c3["t_int"] * 1e3 == pytest.approx(5.170, rel=1e-3)
    assert c3["t_fp"] * 1e3 == pytest.approx(5.083, rel=1e-3)
    c4 = roofline("rademacher", "f32", 10000, 5000, 2_000_000, 1_811_677, 6544, 1965)
    assert c4["bound"] == "fp32_pipe" and c4["t_roof"] * 1e3 == pytest.approx(0.5373, rel=1e-3)
    c5 = roofline("rademacher", "f64", 2000, 1000, 50_000_000, 50_000_000, 6544, 1965)
    rep = roofline_report(c5, 7.238e-3, "f64", 6544, 1965)
    assert rep["bound"] == "fp64_pipe" and rep["frac"] == pytest.approx(0.742, abs=1e-3)
    assert rep["achieved"] == pytest.approx(2 * 2000 * 50e6 / 7.238e-3 / 1e12)
    c1 = roofline("rademacher", "f64", 1000, 500, 10_000, 9_505, 6544, 1965)
    assert c1["bound"] == "hbm"


def test_gpus_n_relaunches_under_torchrun(monkeypatch):
    # `bench.py --gpus N` outside torchrun starts N ranks itself on 127.0.0.1 with the same arguments
    seen = {}

    class _R:
        returncode = 0

    def fake_run(cmd, *a, **k):
        seen["cmd"] = cmd
        return _R()
    monkeypatch.setattr(bench.subprocess, "run", fake_run)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3"])
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    assert bench.main() == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "--master-addr=127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "4", "--steps", "3"]


class _FakePlan:
    def __init__(self, name):
        self.name = name

    def kernel_name(self, dist):
        return self.name


def test_launch_count_per_kernel_family():
    f4 = _FakePlan("sk_rad_f4_kernel (tcgen05 kind::mxf4) + sk_rad_kernel<double>")
    # tensor-core kernel + IEEE fix-up, + the zeroing kernel when the last wave was split along K
    assert bench.launches_per_apply(f4, "rademacher", {"n_items_rad": 0, "n_items_pair": 9, "n_items_f4": 3000,
                                                       "n_items_f4_split": 80}) == 3
    assert bench.launches_per_apply(f4, "rademacher", {"n_items_rad": 0, "n_items_pair": 9, "n_items_f4": 2960,
                                                       "n_items_f4_split": 0}) == 2
    assert bench.launches_per_apply(f4, "rademacher", {"n_items_rad": 5, "n_items_pair": 9, "n_items_f4": 3000,
                                                       "n_items_f4_split": 80}) == 4
    assert bench.launches_per_apply(f4, "rademacher", {"n_items_rad": 5, "n_items_pair": 9, "n_items_f4": 0}) == 1
    f32 = _FakePlan("sk_rad_kernel<float>")
    assert bench.launches_per_apply(f32, "rademacher", {"n_items_rad": 5, "n_items_pair": 9, "n_items_f4": 0}) == 2
    simt = _FakePlan("sk_pair_kernel<uniform, double>")
    assert bench.launches_per_apply(simt, "uniform", {"n_items_rad": 1, "n_items_pair": 10, "n_items_jki": 0}) == 1
    assert bench.launches_per_apply(simt, "uniform", {"n_items_rad": 0, "n_items_pair": 0, "n_items_jki": 0}) == 0
    jki = _FakePlan("sk_jki_kernel<gaussian, double> (Algorithm 4)")
    assert bench.launches_per_apply(jki, "gaussian", {"n_items_rad": 1, "n_items_pair": 10, "n_items_jki": 7}) == 3


def test_traffic_lookup_matches_the_committed_capture():
    path = os.path.join(ROOT, "profiles", "traffic.json")
    with open(path) as f:
        t = json.load(f)
    v = bench.load_profile_traffic("c5", "sk_rad_f4_kernel (tcgen05 kind::mxf4)")
    assert v == t["c5"]["sk_rad_f4_kernel"]
    vp = bench.load_profile_traffic("c5", "sk_rad_f4p_kernel (tcgen05 kind::mxf4, persistent)")
    assert vp == t["c5"]["sk_rad_f4p_kernel"]
    # both tensor-core kernels read A once: DRAM traffic within 2% (per-item) / 3% (persistent, whose
    # scan warp reads the next item's column shortly before the loader does)
    alg = algorithmic_bytes(2000, 1000, 50_000_000, 8)
    assert abs(v - alg) / alg < 0.02
    assert abs(vp - alg) / alg < 0.03


def test_metric_and_bytes_arithmetic():
    # 2 d nnz / t and A-once + Â-once bytes
    assert gflops(2000, 50_000_000, 1.0) == pytest.approx(200.0)
    assert algorithmic_bytes(2000, 1000, 50_000_000, 8) == 8 * 1001 + 12 * 50_000_000 + 8 * 2000 * 1000
