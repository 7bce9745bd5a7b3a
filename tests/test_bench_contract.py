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


def test_alu_peaks_from_unit_counts():
    # 148 SMs x {64 fp64, 128 fp32} lanes x 2 flop x clock
    assert bench.alu_peak_tflops("f64", 1965.0) == pytest.approx(148 * 64 * 2 * 1.965e9 / 1e12)
    assert bench.alu_peak_tflops("f32", 1000.0) == pytest.approx(148 * 128 * 2 * 1e9 / 1e12)


class _FakePlan:
    def __init__(self, name):
        self.name = name

    def kernel_name(self, dist):
        return self.name


def test_launch_count_includes_the_split_zeroing_kernel():
    base = {"n_items_rad": 10, "n_items_pair": 10}
    f4 = _FakePlan("sk_rad_f4_kernel (tcgen05 kind::mxf4)")
    assert bench.launches_per_apply(f4, "rademacher", dict(base, n_items_f4_split=0)) == 1
    assert bench.launches_per_apply(f4, "rademacher", dict(base, n_items_f4_split=316)) == 2
    simt = _FakePlan("sk_pair_kernel<uniform, double>")
    assert bench.launches_per_apply(simt, "uniform", dict(base, n_items_f4_split=316)) == 1
    assert bench.launches_per_apply(simt, "uniform", {"n_items_rad": 0, "n_items_pair": 0}) == 0


def test_traffic_lookup_matches_the_committed_capture():
    path = os.path.join(ROOT, "profiles", "traffic.json")
    with open(path) as f:
        t = json.load(f)
    v = bench.load_profile_traffic("c5", "sk_rad_f4_kernel (tcgen05 kind::mxf4)")
    assert v == t["c5"]["sk_rad_f4_kernel"]
    # the headline kernel reads A once: DRAM traffic within 2% of the algorithmic bytes
    alg = algorithmic_bytes(2000, 1000, 50_000_000, 8)
    assert abs(v - alg) / alg < 0.02


def test_metric_and_bytes_arithmetic():
    # 2 d nnz / t and A-once + Â-once bytes
    assert gflops(2000, 50_000_000, 1.0) == pytest.approx(200.0)
    assert algorithmic_bytes(2000, 1000, 50_000_000, 8) == 8 * 1001 + 12 * 50_000_000 + 8 * 2000 * 1000
