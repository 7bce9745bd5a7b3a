"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (north star, DESIGN.md §"Parity"):
  * S entries: bit-exact for ±1 and uniform (fp64 and fp32); Gaussian |ΔS| <= 1e-14 |S|.
  * Â: |Â_gpu - Â_oracle| <= 1e-12 · B (fp64) or 2e-5 · B (fp32), B = |S|·|A| elementwise;
    entries with B = 0 must be exactly ±0.
"""
import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-12, "f32": 2e-5}


@pytest.fixture(scope="module")
def sk():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    from paper_2310_15419_b200 import sketch
    sketch.load_library()
    return sketch


def _dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _gpu_sketch(sk, A, d, dist, seed):
    plan = sk.Plan(_dev(A.colptr), _dev(A.rowidx), d, A.m,
                   "f32" if A.vals.dtype == np.float32 else "f64", row_offset=A.row_offset)
    out = plan.apply(_dev(A.vals), seed, dist)
    import torch
    torch.cuda.synchronize()
    res = out.T.double().cpu().numpy()
    plan.close()
    return res


def _check(got, ref, bound, tol):
    err = np.abs(got - ref)
    ok = err <= tol * bound
    zero = bound == 0
    assert np.all(got[zero] == 0), "entries with B = 0 must be exactly zero"
    if not np.all(ok):
        i = np.unravel_index(np.argmax(err / np.maximum(bound, 1e-300)), err.shape)
        raise AssertionError(f"max rel err {(err / np.maximum(bound, 1e-300)).max():.3e} at {i}")


# ------------------------------------------------------------------- S entries

FILL_CASES = [
    # (i0, i1, j0, j1): edges of Philox blocks (127/128), ragged tails, large j (j_hi != 0)
    (0, 300, 0, 5),
    (100, 389, 7, 9),
    (127, 129, 0, 3),
    (0, 1, 0, 1),
    (1000, 1031, 2**32 - 2, 2**32 + 3),
    (0, 257, 49_999_998, 50_000_000),
]


@pytest.mark.parametrize("dist", ["rademacher", "uniform", "gaussian", "uniform24"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_fill_s_matches_oracle(sk, dist, dtype):
    for (i0, i1, j0, j1) in FILL_CASES:
        for seed in (0, 4, 2**63 + 12345):
            got = sk.sketch_fill_s(seed, dist, i0, i1, j0, j1, dtype).T.double().cpu().numpy()
            ref = oracle.fill_s(seed, dist, i0, i1, j0, j1, dtype=dtype)
            if dist == "gaussian":
                assert np.all(np.abs(got - ref) <= 1e-14 * np.abs(ref)), (dtype, i0, j0, seed)
            else:
                assert np.array_equal(got, ref), (dist, dtype, i0, j0, seed)


def test_gaussian_entries_dense(sk):
    # 2M Gaussian entries (own fp64 log / sincos, philox.cuh) against the libm-based oracle: the
    # whole (u1, u2) range is exercised, including u1 near 1 (rho -> 0) and theta near k pi/2
    seed, i1, j0, j1 = 2, 4096, 123_456, 123_456 + 512
    got = sk.sketch_fill_s(seed, "gaussian", 0, i1, j0, j1).T.cpu().numpy()
    ref = oracle.fill_s(seed, "gaussian", 0, i1, j0, j1)
    rel = np.abs(got - ref) / np.abs(ref)
    assert np.all(rel <= 1e-14), float(rel.max())
    assert float(np.median(rel)) < 2.3e-16         # typically within an ulp


def test_fill_s_matches_curand_philox(sk):
    # Independent implementation: cuRAND's Philox4_32_10 with curand_init(seed, j, 4q) gives
    # the block (q, 0, j_lo, j_hi); its bits, read as ±1, must equal our S.
    import torch
    from torch.utils.cpp_extension import load_inline
    src = r"""
#include <curand_kernel.h>
__global__ void k(unsigned long long seed, long long j0, int nq, int nj, unsigned* out) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nq * nj) return;
  int q = idx % nq; long long j = j0 + idx / nq;
  curandStatePhilox4_32_10_t st;
  curand_init(seed, (unsigned long long)j, 4ull * q, &st);
  uint4 x = curand4(&st);
  out[4*idx+0] = x.x; out[4*idx+1] = x.y; out[4*idx+2] = x.z; out[4*idx+3] = x.w;
}
torch::Tensor run(long long seed, long long j0, int nq, int nj) {
  auto out = torch::empty({nq * nj * 4}, torch::dtype(torch::kInt32).device(torch::kCUDA));
  k<<<(nq*nj + 127)/128, 128>>>((unsigned long long)seed, j0, nq, nj, (unsigned*)out.data_ptr());
  return out;
}
"""
    try:
        mod = load_inline("curand_ref", cpp_sources="torch::Tensor run(long long, long long, int, int);",
                          cuda_sources=src, functions=["run"], verbose=False,
                          extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a"])
    except Exception as e:  # pragma: no cover - toolchain issue, not a parity failure
        pytest.skip(f"cannot build cuRAND reference: {e}")
    seed, j0, nq, nj = 987654321, 2**32 - 3, 4, 6
    words = mod.run(seed, j0, nq, nj).cpu().numpy().view(np.uint32).reshape(nj, nq, 4)
    S = sk.sketch_fill_s(seed, "rademacher", 0, 128 * nq, j0, j0 + nj).cpu().numpy()  # (nj, rows)
    for jj in range(nj):
        for q in range(nq):
            for t in range(4):
                bits = (int(words[jj, q, t]) >> np.arange(32)) & 1
                expect = np.where(bits == 1, -1.0, 1.0)
                assert np.array_equal(S[jj, 128 * q + 32 * t: 128 * q + 32 * t + 32], expect)
    # and the oracle's Philox agrees with cuRAND word for word
    for jj in range(nj):
        for q in range(nq):
            j = j0 + jj
            ref = oracle.philox4x32_10([q, 0, j & 0xFFFFFFFF, j >> 32], [seed & 0xFFFFFFFF, seed >> 32])
            assert tuple(int(w) for w in words[jj, q]) == ref


# ------------------------------------------------------------------- Â = S·A, small / edge

SMALL = [
    # (name, A builder, d)
    ("tiny", lambda: workloads.random_csc(300, 7, 5, seed=1), 70),
    ("ragged_d", lambda: workloads.random_csc(5000, 40, 33, seed=2), 1000),
    ("multi_tile_d", lambda: workloads.random_csc(20000, 30, 50, seed=3), 4500),
    ("d1", lambda: workloads.random_csc(1000, 9, 17, seed=4), 1),
    ("empty_cols", lambda: workloads.random_csc(3000, 12, [0, 5, 0, 0, 64, 1, 0, 33, 0, 2, 0, 100], seed=5), 300),
    ("long_and_short", lambda: workloads.random_csc(200000, 24, [20000] + [10] * 23, seed=6), 1100),
    ("unsorted_dups", lambda: workloads.random_csc(500, 10, 40, seed=7, sorted_rows=False, duplicates=True), 129),
    ("abnormal_A_dense_rows", lambda: workloads.abnormal("A", 10000, 60, 3000, seed=8), 257),
    ("abnormal_C_dense_cols", lambda: workloads.abnormal("C", 2000, 50, 3000, seed=9), 513),
]


@pytest.mark.parametrize("dist", ["rademacher", "uniform", "gaussian", "uniform24"])
@pytest.mark.parametrize("case", SMALL, ids=[c[0] for c in SMALL])
def test_sketch_matches_oracle_small(sk, dist, case):
    name, build, d = case
    A = build()
    seed = 77
    got = _gpu_sketch(sk, A, d, dist, seed)
    ref, B = oracle.sketch(seed, dist, d, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=8)
    _check(got, ref, B, TOL["f64"])


@pytest.mark.parametrize("path", ["fp4", "simt"])
def test_rad_f64_kernel_paths(sk, path):
    # both ±1 fp64 kernel selections (tensor cores + SIMT for short columns, SIMT only) meet the fp64 bar on
    # the edge cases: ragged d and tiles, empty and single-nonzero columns, a column that is long
    # relative to the rest, unsorted rows with duplicates, explicit zeros and huge / tiny values
    try:
        sk.set_rad_f64_path(path)
        # (columns of 896 / 1280 .. 131071 nonzeros run on the tensor cores, the others on the SIMT kernel)
        cases = [workloads.random_csc(50000, 40, 1300, seed=2),
                 workloads.random_csc(30000, 12, [0, 500, 0, 0, 1640, 1, 0, 3300, 0, 2, 0, 1279], seed=5),
                 workloads.random_csc(200000, 24, [20000] + [10] * 23, seed=6),
                 workloads.random_csc(5000, 10, 1400, seed=7, sorted_rows=False, duplicates=True)]
        wide = workloads.random_csc(40000, 6, 1700, seed=17)
        wide.vals = wide.vals * np.logspace(-200, 200, wide.nnz)       # dynamic range per column
        wide.vals[::7] = 0.0
        cases.append(wide)
        for A, d in zip(cases, [1000, 300, 1100, 129, 2050]):
            got = _gpu_sketch(sk, A, d, "rademacher", 31)
            ref, B = oracle.sketch(31, "rademacher", d, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=8)
            _check(got, ref, B, TOL["f64"])
    finally:
        sk.set_rad_f64_path("fp4")


@pytest.mark.parametrize("path", ["fp4", "simt"])
def test_nan_poisons_only_its_column(sk, path):
    # a NaN value makes its whole column NaN (NaN * ±1 = NaN in every row, as in the oracle); the
    # other columns are unaffected.  (fmax-based column scans would drop the NaN: the tensor-core
    # kernels take max |a| on the IEEE bit patterns, NaN > Inf > finite.)
    A = workloads.random_csc(50000, 6, 1500, seed=41)
    A.vals[A.colptr[2] + 5] = np.nan
    try:
        sk.set_rad_f64_path(path)
        for dist in ("rademacher", "uniform", "gaussian"):
            got = _gpu_sketch(sk, A, 700, dist, 3)
            ref, B = oracle.sketch(3, dist, 700, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=8)
            assert np.isnan(got[:, 2]).all() and np.isnan(ref[:, 2]).all()
            keep = [0, 1, 3, 4, 5]
            _check(got[:, keep], ref[:, keep], B[:, keep], TOL["f64"])
    finally:
        sk.set_rad_f64_path("fp4")


def test_rad_f32_edge_cases(sk):
    # the ±1 fp32 kernel on the edge cases: ragged d and item tails (d not a multiple of 128 or
    # 2048), empty / single / long columns, chunk tails (lengths not multiples of 32 or 4),
    # unsorted rows with duplicates, d = 1
    f32 = np.float32
    cases = [(workloads.random_csc(50000, 40, 300, seed=2, dtype=f32), 1000),
             (workloads.random_csc(30000, 12, [0, 500, 0, 0, 641, 1, 0, 3303, 0, 2, 0, 99], seed=5, dtype=f32), 2100),
             (workloads.random_csc(5000, 10, 37, seed=7, sorted_rows=False, duplicates=True, dtype=f32), 129),
             (workloads.random_csc(4000, 7, 45, seed=9, dtype=f32), 1),
             (workloads.random_csc(200000, 3, [20000, 3, 7], seed=6, dtype=f32), 4097)]
    for A, d in cases:
        got = _gpu_sketch(sk, A, d, "rademacher", 13)
        ref, B = oracle.sketch(13, "rademacher", d, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=8)
        _check(got, ref, B, TOL["f32"])


INF_DISTS = [("rademacher", "f64", "fp4"), ("rademacher", "f64", "simt"), ("rademacher", "f32", "fp4"),
             ("uniform", "f64", "fp4"), ("gaussian", "f64", "fp4"), ("uniform24", "f32", "fp4"),
             ("uniform", "f64", "jki"), ("gaussian", "f32", "jki")]


@pytest.mark.parametrize("dist,dtype,path", INF_DISTS, ids=["-".join(x) for x in INF_DISTS])
def test_infinite_values_follow_ieee(sk, dist, dtype, path):
    # ±Inf values give the IEEE sum on every path (the tensor-core kernel used to write NaN):
    # column 1 holds one +Inf (every row ±Inf by its S sign), column 3 a +Inf and a -Inf (rows where the
    # two terms have opposite signs are NaN, the others ±Inf), column 4 an Inf and a NaN (all NaN); the
    # other columns stay finite and within the parity bar.  Columns are long enough (2100) for the
    # tensor-core kernel.
    import torch
    npdt = np.float32 if dtype == "f32" else np.float64
    A = workloads.random_csc(60000, 6, 2100, seed=43, dtype=npdt)
    A.vals[A.colptr[1] + 17] = np.inf
    A.vals[A.colptr[3] + 5] = np.inf
    A.vals[A.colptr[3] + 900] = -np.inf
    A.vals[A.colptr[4] + 3] = -np.inf
    A.vals[A.colptr[4] + 1000] = np.nan
    d = 900
    try:
        if path == "simt":
            sk.set_rad_f64_path("simt")
        plan = sk.Plan(_dev(A.colptr), _dev(A.rowidx), d, A.m, dtype, jki=path == "jki")
        if path == "fp4" and dist == "rademacher" and dtype == "f64":
            assert plan.stats()["n_cols_f4"] == 6
        got = plan.apply(_dev(A.vals), 3, dist).T.double().cpu().numpy()
        torch.cuda.synchronize()
        plan.close()
    finally:
        sk.set_rad_f64_path("fp4")
    ref, B = oracle.sketch(3, dist, d, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=8)
    for k in (1, 3, 4):
        assert np.array_equal(np.isnan(got[:, k]), np.isnan(ref[:, k])), k
        fin = ~np.isnan(ref[:, k])
        assert np.all(np.isinf(ref[fin, k])) and np.array_equal(got[fin, k], ref[fin, k]), k
    assert np.isnan(ref[:, 3]).any() and (~np.isnan(ref[:, 3])).any()
    keep = [0, 2, 5]
    _check(got[:, keep], ref[:, keep], B[:, keep], TOL[dtype])


def test_f4_last_wave_split_along_k(sk):
    # 160 one-item columns on 148 SMs: the plan splits the last wave (here every tensor-core item)
    # into two K halves that add into zeroed rows (0 + a + b rounds the same in either order).  Short
    # columns go to the SIMT kernel, results match the oracle, and two runs are bit-identical.
    import torch
    lens = [2100] * 160
    lens[7], lens[50], lens[51] = 40, 127, 129
    A = workloads.random_csc(60000, 160, lens, seed=23)
    plan = sk.Plan(_dev(A.colptr), _dev(A.rowidx), 700, A.m, "f64")
    try:
        st = plan.stats()
        assert st["n_cols_f4"] == 157 and st["n_items_rad"] > 0
        if torch.cuda.get_device_properties(0).multi_processor_count == 148:
            assert st["n_items_f4_split"] == 2 * 157
        assert "sk_rad_f4" in plan.kernel_name("rademacher")
        vals = _dev(A.vals)
        o1 = plan.apply(vals, 3, "rademacher").T.cpu().numpy()
        o2 = plan.apply(vals, 3, "rademacher").T.cpu().numpy()
        assert np.array_equal(o1, o2)
        ref, B = oracle.sketch(3, "rademacher", 700, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=8)
        _check(o1, ref, B, TOL["f64"])
    finally:
        plan.close()


def test_f4_long_columns_next_to_tensor_columns(sk):
    # the tensor-core path is chosen per column, not per matrix: a column longer than 131071 nonzeros
    # (the exact-accumulation bound) and short ones run on the SIMT kernel, concurrently on a side
    # stream, while every other column stays on sk_rad_f4_kernel; results match the oracle and two
    # runs are bit-identical
    import torch
    lens = [300000, 131072, 131071, 3000, 1279, 1280, 700, 90]   # (one wave of items: threshold 1280)
    A = workloads.random_csc(400000, len(lens), lens, seed=29)
    plan = sk.Plan(_dev(A.colptr), _dev(A.rowidx), 1300, A.m, "f64")
    try:
        st = plan.stats()
        assert st["n_cols_f4"] == 3 and st["n_items_rad"] > 0, st
        assert "sk_rad_f4" in plan.kernel_name("rademacher")
        vals = _dev(A.vals)
        o1 = plan.apply(vals, 6, "rademacher").T.cpu().numpy()
        o2 = plan.apply(vals, 6, "rademacher").T.cpu().numpy()
        torch.cuda.synchronize()
        assert np.array_equal(o1, o2)
    finally:
        plan.close()
    ref, B = oracle.sketch(6, "rademacher", 1300, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=16)
    _check(o1, ref, B, TOL["f64"])


@pytest.mark.parametrize("d", [2000, 700, 2500])
def test_f4_persistent_kernel_matches_per_item_kernel(sk, d):
    # the persistent tensor-core kernel (one CTA per SM walking ~4 items each here: 600+ items of
    # 6 / 6 / 4 or 6 or 5 / 5 / 5 / 5 row tiles, K-split last-wave halves, a NaN column, a column
    # exactly at the threshold) computes every item with the same arithmetic as the one-CTA-per-item
    # kernel: bit-identical results, and both match the oracle
    import torch
    rng = np.random.default_rng(d)
    lens = [int(x) for x in rng.integers(1280, 9000, size=211)]
    lens[3] = 1280
    A = workloads.random_csc(50000, len(lens), lens, seed=d + 1)
    A.vals[A.colptr[10] + 5] = np.nan
    outs = {}
    try:
        for mode in ("off", "on"):
            sk.set_f4_persistent(mode)
            plan = sk.Plan(_dev(A.colptr), _dev(A.rowidx), d, A.m, "f64")
            try:
                st = plan.stats()
                assert st["n_cols_f4"] == len(lens) and st["f4_persistent"] == (mode == "on")
                assert ("sk_rad_f4p_kernel" in plan.kernel_name("rademacher")) == (mode == "on")
                outs[mode] = plan.apply(_dev(A.vals), 12, "rademacher").T.cpu().numpy()
                torch.cuda.synchronize()
            finally:
                plan.close()
    finally:
        sk.set_f4_persistent("auto")
    assert np.array_equal(outs["on"], outs["off"], equal_nan=True)
    ref, B = oracle.sketch(12, "rademacher", d, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=16)
    assert np.all(np.isnan(outs["on"][:, 10])) and np.all(np.isnan(ref[:, 10]))
    keep = [k for k in range(A.n) if k != 10]
    _check(outs["on"][:, keep], ref[:, keep], B[:, keep], TOL["f64"])


@pytest.mark.parametrize("d", [100, 129, 768])
def test_f4_persistent_kernel_edge_shapes(sk, d):
    # persistent kernel with 1-tile items (10 idle S warps per item: the digit warps arrive for them),
    # a ragged last tile, columns at the thresholds (896, 131071), lengths that fill whole K-steps
    # (no padding) and lengths one past them
    import torch
    lens = [896, 131071, 1024, 1025, 4096, 4097, 963] + [900 + 7 * k for k in range(200)]
    A = workloads.random_csc(400000, len(lens), lens, seed=61)
    plan = sk.Plan(_dev(A.colptr), _dev(A.rowidx), d, A.m, "f64")
    try:
        st = plan.stats()
        assert st["f4_persistent"] == 1 and st["n_cols_f4"] == len(lens), st
        got = plan.apply(_dev(A.vals), 31, "rademacher").T.cpu().numpy()
        torch.cuda.synchronize()
    finally:
        plan.close()
    ref, B = oracle.sketch(31, "rademacher", d, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=16)
    _check(got, ref, B, TOL["f64"])


def test_f4_persistent_kernel_with_row_offset(sk):
    # a row shard (global row keys j + row_offset > 2^32) on the persistent kernel: its read-out
    # removes the padding's share of the ones row with S[i, row_offset], so a wrong offset there
    # would show in every column whose length is not a multiple of 64
    import torch
    rng = np.random.default_rng(5)
    lens = [int(x) for x in rng.integers(900, 4000, size=180)]
    A = workloads.random_csc(70000, len(lens), lens, seed=55)
    A.row_offset = (1 << 32) + 777
    try:
        sk.set_f4_persistent("on")
        plan = sk.Plan(_dev(A.colptr), _dev(A.rowidx), 1000, A.m, "f64", row_offset=A.row_offset)
        try:
            st = plan.stats()
            assert st["f4_persistent"] == 1 and st["n_cols_f4"] == len(lens)
            got = plan.apply(_dev(A.vals), 29, "rademacher").T.cpu().numpy()
            torch.cuda.synchronize()
        finally:
            plan.close()
    finally:
        sk.set_f4_persistent("auto")
    ref, B = oracle.sketch(29, "rademacher", 1000, A.m, A.n, A.colptr, A.rowidx, A.vals, row_offset=A.row_offset,
                           threads=16)
    _check(got, ref, B, TOL["f64"])


def test_f4_persistent_selection(sk):
    # the plan picks the persistent kernel when there is more than one wave of tensor-core items (600
    # items here, c5's 3188) and one CTA per item for a single wave (80 items)
    short = workloads.random_csc(100000, 300, 6000, seed=3)
    long_ = workloads.random_csc(200000, 40, 40000, seed=4)
    for A, want in ((short, 1), (long_, 0)):
        plan = sk.Plan(_dev(A.colptr), _dev(A.rowidx), 1000, A.m, "f64")
        try:
            assert plan.stats()["f4_persistent"] == want
        finally:
            plan.close()


def test_apply_captures_into_cuda_graph(sk):
    # sketch_apply is stream-ordered all the way down (kernels, the library pool's scratch, the
    # persistent kernel's item counter, the side stream of the SIMT columns joined by events), so a
    # CUDA graph captures it and replays it with the eager results, bit for bit: ±1 with tensor-core
    # (persistent) and SIMT columns, uniform Algorithm 3, Gaussian Algorithm 4
    import torch
    lens = [3000] * 300 + [50, 700, 0, 200000]
    A = workloads.random_csc(300000, len(lens), lens, seed=41)
    R = workloads.abnormal_paper("A", m=20000, n=70, seed=1)
    cases = [(A, "rademacher", False, 600), (A, "uniform", False, 600), (R, "gaussian", True, 700)]
    for M, dist, jki, d in cases:
        plan = sk.Plan(_dev(M.colptr), _dev(M.rowidx), d, M.m, "f64", jki=jki)
        try:
            if dist == "rademacher":
                st = plan.stats()
                assert st["n_items_f4"] > 0 and st["n_items_rad"] > 0
            if jki:
                sk.set_pair_path("jki")
            vals = _dev(M.vals)
            eager = plan.apply(vals, 17, dist).clone()
            out = torch.empty_like(eager)
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                plan.apply(vals, 17, dist, out=out)          # warm-up on the capture stream
            torch.cuda.current_stream().wait_stream(s)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                plan.apply(vals, 17, dist, out=out)
            for _ in range(2):
                out.zero_()
                g.replay()
                torch.cuda.synchronize()
                assert torch.equal(out, eager), (dist, float((out - eager).abs().max()))
        finally:
            sk.set_pair_path("auto")
            plan.close()


@pytest.mark.parametrize("case", range(16))
def test_randomized_shapes_match_oracle(sk, case):
    # seeded random shapes through the default kernel selection: m, n, column lengths (empty,
    # short, >= 1280 so the tensor-core path is eligible, occasionally one very long column), d
    # (ragged, tiny, > 2048), dtype, distribution and a nonzero row offset
    rng = np.random.default_rng(1000 + case)
    m = int(rng.integers(1, 60000))
    n = int(rng.integers(1, 24))
    kind = case % 4
    if kind == 0:
        lens = rng.integers(0, 40, n)
    elif kind == 1:
        lens = rng.integers(1280, 2000, n)
    elif kind == 2:
        lens = rng.integers(0, 900, n)
        lens[int(rng.integers(0, n))] = min(m, 5000)
    else:
        lens = rng.integers(1200, 1400, n)
    lens = [int(min(L, m)) for L in lens]
    d = int(rng.choice([1, 2, 127, 129, 700, 1025, 2049, int(rng.integers(1, 2200))]))
    dtype = np.float32 if case % 3 == 2 else np.float64
    dist = ["rademacher", "uniform", "gaussian", "uniform24"][case % 4 if case % 5 else 0]
    A = workloads.random_csc(m, n, lens, seed=case, dtype=dtype, sorted_rows=bool(case % 2),
                             duplicates=case % 7 == 3)
    A.row_offset = int(rng.integers(0, 1 << 20))
    got = _gpu_sketch(sk, A, d, dist, 17 + case)
    ref, B = oracle.sketch(17 + case, dist, d, A.m, A.n, A.colptr, A.rowidx, A.vals, row_offset=A.row_offset,
                           threads=8)
    _check(got, ref, B, TOL["f32" if dtype == np.float32 else "f64"])


@pytest.mark.parametrize("dist,dtype", [("rademacher", "f64"), ("rademacher", "f32"), ("uniform", "f64"),
                                        ("gaussian", "f64")])
def test_repeated_runs_are_bit_identical(sk, dist, dtype):
    # race check without a sanitizer: 25 back-to-back applies of the same plan on a matrix whose
    # schedule uses every stage of the pipelines (long columns, ragged tail, K-split last wave)
    # must give bit-identical outputs (all reductions have a fixed order; the tensor-core path
    # accumulates integers)
    import torch
    A = workloads.random_csc(400000, 170, 1500, seed=31, dtype=np.float32 if dtype == "f32" else np.float64)
    plan = sk.Plan(_dev(A.colptr), _dev(A.rowidx), 1900, A.m, dtype)
    try:
        vals = _dev(A.vals)
        first = plan.apply(vals, 8, dist).clone()
        for _ in range(24):
            assert torch.equal(plan.apply(vals, 8, dist), first)
    finally:
        plan.close()


@pytest.mark.parametrize("path", ["fp4", "simt"])
def test_extreme_value_scales(sk, path):
    # columns whose values are all subnormal, all near the top of the fp64 range, or mix both with
    # exact zeros: the tensor-core paths scale each column by 2^(61-E) in two exact factors
    A = workloads.random_csc(30000, 5, 1400, seed=41)
    v = A.vals.copy()
    s = [slice(A.colptr[k], A.colptr[k + 1]) for k in range(5)]
    v[s[0]] *= 1e-310                                  # subnormal
    v[s[1]] *= 1e300                                   # huge (|Â| stays < 1e308 for 1400 terms)
    v[s[2]] = np.where(np.arange(1400) % 2 == 0, v[s[2]] * 1e-300, v[s[2]] * 1e200)
    v[s[3]] = 0.0                                      # all explicit zeros
    v[s[4]][::3] = 0.0
    A.vals = v
    try:
        sk.set_rad_f64_path(path)
        got = _gpu_sketch(sk, A, 600, "rademacher", 9)
        ref, B = oracle.sketch(9, "rademacher", 600, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=8)
        assert np.all(np.isfinite(got))
        _check(got, ref, B, TOL["f64"])
    finally:
        sk.set_rad_f64_path("fp4")


def test_kernel_names_report_the_path(sk):
    A = workloads.random_csc(10000, 4, 3000, seed=1)
    try:
        for path, tag in (("fp4", "mxf4"), ("simt", "sk_rad_kernel<double>")):
            sk.set_rad_f64_path(path)
            plan = sk.Plan(_dev(A.colptr), _dev(A.rowidx), 300, A.m, "f64")
            assert tag in plan.kernel_name("rademacher")
            assert "uniform" in plan.kernel_name("uniform") and "gaussian" in plan.kernel_name("gaussian")
            plan.close()
        A32 = workloads.random_csc(10000, 4, 300, seed=1, dtype=np.float32)
        plan32 = sk.Plan(_dev(A32.colptr), _dev(A32.rowidx), 300, A32.m, "f32")
        assert "sk_rad_kernel<float>" in plan32.kernel_name("rademacher")
        plan32.close()
    finally:
        sk.set_rad_f64_path("fp4")


@pytest.mark.parametrize("dist", ["rademacher", "uniform", "gaussian", "uniform24"])
def test_sketch_f32_matches_oracle(sk, dist):
    A = workloads.random_csc(20000, 25, 120, seed=10, dtype=np.float32)
    got = _gpu_sketch(sk, A, 2100, dist, 5)
    ref, B = oracle.sketch(5, dist, 2100, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=8)
    _check(got, ref, B, TOL["f32"])


def test_exact_cases_bitwise(sk):
    # ±1 S with small-integer A: every partial sum is exact, so GPU == oracle bit for bit in
    # any summation order; A = I gives Â = S exactly.
    A = workloads.random_csc(4000, 20, 300, seed=11, values="smallint")
    got = _gpu_sketch(sk, A, 1500, "rademacher", 3)
    ref, _ = oracle.sketch(3, "rademacher", 1500, A.m, A.n, A.colptr, A.rowidx, A.vals)
    assert np.array_equal(got, ref)
    m = 50
    I = workloads.CSC(m, m, np.arange(m + 1, dtype=np.int64), np.arange(m, dtype=np.int32), np.ones(m))
    for dist in ("rademacher", "uniform", "gaussian"):
        got = _gpu_sketch(sk, I, 300, dist, 9)
        ref = oracle.fill_s(9, dist, 0, 300, 0, m)
        if dist == "gaussian":
            assert np.all(np.abs(got - ref) <= 1e-14 * np.abs(ref))
        else:
            assert np.array_equal(got, ref)


def test_row_offset_and_shards(sk):
    # global-j keys: a shard planned with row_offset reproduces its slice of the full sketch,
    # including row offsets past 2^32 (high counter word)
    A = workloads.random_csc(30000, 16, 200, seed=12)
    full = _gpu_sketch(sk, A, 700, "rademacher", 21)
    tot = np.zeros_like(full)
    for g in range(3):
        Ag = workloads.shard_csc(A, 3, g)
        tot += _gpu_sketch(sk, Ag, 700, "rademacher", 21)
    ref, B = oracle.sketch(21, "rademacher", 700, A.m, A.n, A.colptr, A.rowidx, A.vals)
    _check(full, ref, B, 1e-12)
    _check(tot, ref, B, 1e-12)
    Ab = workloads.random_csc(1000, 5, 30, seed=13)
    Ab.row_offset = 2**32 + 17
    got = _gpu_sketch(sk, Ab, 300, "uniform", 1)
    ref, B = oracle.sketch(1, "uniform", 300, Ab.m, Ab.n, Ab.colptr, Ab.rowidx, Ab.vals,
                           row_offset=Ab.row_offset)
    _check(got, ref, B, 1e-12)


@pytest.mark.parametrize("dist", ["rademacher", "uniform", "gaussian"])
def test_col_shards_and_overlapped_row_reduce(sk, dist):
    # column shards: nnz-balanced column blocks sketched independently are the
    # columns of the full sketch, bit for bit (every column is computed the same way); and the
    # row-sharded driver with the reduction overlapped per column group gives the plain result
    # (Algorithm 3 for all: a column's bits then depend only on its own nonzeros and the tile shape;
    # the automatic choice may pick Algorithm 4 for the full matrix but not for a shard, which moves
    # the rounding within the parity bar -- checked below against the oracle)
    import torch
    from paper_2310_15419_b200.distributed import balanced_col_shards, sketch_row_sharded_overlapped
    A = workloads.random_csc(40000, 30, [300 + 37 * k for k in range(30)], seed=31)
    d = 900
    ref, B = oracle.sketch(8, dist, d, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=8)
    _check(_gpu_sketch(sk, A, d, dist, 8), ref, B, TOL["f64"])
    try:
        sk.set_pair_path("kji")
        full = _gpu_sketch(sk, A, d, dist, 8)
        b = balanced_col_shards(A.colptr, 3)
        blocks = [_gpu_sketch(sk, workloads.col_slice(A, b[g], b[g + 1]), d, dist, 8) for g in range(3)]
        assert np.array_equal(np.concatenate(blocks, axis=1), full)
        out = sketch_row_sharded_overlapped(A.colptr, _dev(A.colptr), _dev(A.rowidx), _dev(A.vals), d, A.m, 0, 8,
                                            dist, groups=4)
        torch.cuda.synchronize()
        assert np.array_equal(out.T.cpu().numpy(), full)
    finally:
        sk.set_pair_path("auto")
    _check(full, ref, B, TOL["f64"])


def test_degenerate_shapes(sk):
    import torch
    # n = 0, nnz = 0 (all-empty columns -> zeros written over garbage)
    A = workloads.CSC(100, 4, np.zeros(5, np.int64), np.zeros(0, np.int32), np.zeros(0))
    plan = sk.Plan(_dev(A.colptr), torch.zeros(0, dtype=torch.int32, device="cuda"), 130, 100)
    out = torch.full((4, 130), float("nan"), dtype=torch.float64, device="cuda")
    plan.apply(torch.zeros(0, dtype=torch.float64, device="cuda"), 1, "gaussian", out=out)
    torch.cuda.synchronize()
    assert torch.count_nonzero(out).item() == 0
    A0 = workloads.CSC(10, 0, np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0))
    plan = sk.Plan(_dev(A0.colptr), torch.zeros(0, dtype=torch.int32, device="cuda"), 5, 10)
    assert plan.apply(torch.zeros(0, dtype=torch.float64, device="cuda"), 1, "uniform").shape == (0, 5)


def test_extreme_index_ranges(sk):
    # global rows near 2^31 (m just below the int32 bound, rows at the top of the range, plus a
    # row offset past 2^32 so the Philox counter's high word j >> 32 is nonzero) and a large d
    # (many row tiles: tile indices and Philox block indices q far from 0), on the default paths
    rng = np.random.default_rng(77)
    m = 2**31 - 1
    n = 6
    cols = []
    for k in range(n):
        L = 300 if k % 2 == 0 else 17
        rows = np.sort(rng.choice(np.arange(m - 5000, m, dtype=np.int64), size=L, replace=False))
        cols.append(rows)
    colptr = np.zeros(n + 1, np.int64)
    colptr[1:] = np.cumsum([len(c) for c in cols])
    rowidx = np.concatenate(cols).astype(np.int32)
    vals = rng.standard_normal(int(colptr[-1]))
    A = workloads.CSC(m, n, colptr, rowidx, vals, row_offset=(1 << 32) + 12345)
    for dist, d in (("rademacher", 70001), ("uniform", 9000), ("gaussian", 3001)):
        got = _gpu_sketch(sk, A, d, dist, 5)
        ref, B = oracle.sketch(5, dist, d, A.m, A.n, A.colptr, A.rowidx, A.vals, row_offset=A.row_offset,
                               threads=8)
        _check(got, ref, B, TOL["f64"])


def test_csc_validation_errors(sk):
    import torch
    colptr = _dev(np.array([0, 2, 1, 3], np.int64))
    rows = _dev(np.array([0, 1, 2], np.int32))
    with pytest.raises(sk.SketchError) as e:
        sk.Plan(colptr, rows, 10, 5)
    assert e.value.code == sk.SK_ECSC
    colptr = _dev(np.array([0, 2, 3], np.int64))
    rows = _dev(np.array([0, 5, 2], np.int32))     # row 5 >= m = 5
    with pytest.raises(sk.SketchError) as e:
        sk.Plan(colptr, rows, 10, 5)
    assert e.value.code == sk.SK_ECSC
    rows = _dev(np.array([0, -1, 2], np.int32))
    with pytest.raises(sk.SketchError):
        sk.Plan(colptr, rows, 10, 5)
    del torch


def test_apply_csc_and_host_entry_points(sk):
    import torch
    A = workloads.random_csc(40000, 64, 150, seed=14)
    ref, B = oracle.sketch(8, "rademacher", 1200, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=8)
    out = sk.sketch_apply_csc(8, "rademacher", 1200, A.m, _dev(A.colptr), _dev(A.rowidx), _dev(A.vals))
    torch.cuda.synchronize()
    _check(out.T.cpu().numpy(), ref, B, 1e-12)
    for chunks in (0, 1, 3, 64):
        h = sk.sketch_apply_host(8, "rademacher", 1200, A.m, A.colptr, A.rowidx, A.vals,
                                 pipeline_chunks=chunks)
        _check(h.T, ref, B, 1e-12)
    # pinned host buffers + fp32
    A32 = workloads.random_csc(40000, 33, 90, seed=15, dtype=np.float32)
    ref32, B32 = oracle.sketch(2, "uniform", 900, A32.m, A32.n, A32.colptr, A32.rowidx, A32.vals, threads=8)
    pin = lambda a: torch.from_numpy(a).pin_memory()
    out = torch.empty((A32.n, 900), dtype=torch.float32).pin_memory()
    sk.sketch_apply_host(2, "uniform", 900, A32.m, pin(A32.colptr), pin(A32.rowidx), pin(A32.vals),
                         out=out, pipeline_chunks=4)
    _check(out.numpy().T.astype(np.float64), ref32, B32, 2e-5)


def test_tiling_invariance_of_result(sk):
    # Results must not depend on the schedule beyond rounding order: the same matrix with its
    # columns permuted gives the permuted sketch (different CTA order / shapes).
    A = workloads.random_csc(10000, 30, [5 * (k + 1) for k in range(30)], seed=16)
    got = _gpu_sketch(sk, A, 2500, "gaussian", 4)
    perm = np.random.default_rng(0).permutation(30)
    Ap = A.select_columns(perm)
    gotp = _gpu_sketch(sk, Ap, 2500, "gaussian", 4)
    ref, B = oracle.sketch(4, "gaussian", 2500, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=8)
    _check(got, ref, B, 1e-12)
    _check(gotp, ref[:, perm], B[:, perm], 1e-12)


# ------------------------------------------------------------------- BASELINE.json configs

def _config_parity(sk, name):
    """Full-size config on the GPU in the launch configuration bench.py times (one Plan over the
    whole matrix, one sketch_apply), compared with the oracle on EVERY column."""
    cfg = workloads.CONFIGS[name]
    A = workloads.make_config(name)
    got = _gpu_sketch(sk, A, cfg.d, cfg.dist, cfg.seed)
    assert got.shape == (cfg.d, cfg.n)
    ref, B = oracle.sketch(cfg.seed, cfg.dist, cfg.d, A.m, A.n, A.colptr, A.rowidx, A.vals,
                           threads=oracle.max_threads())
    _check(got, ref, B, TOL[cfg.dtype])
    assert np.all(np.isfinite(got))


def test_config_c1_full(sk):
    _config_parity(sk, "c1")


def test_config_c2_full(sk):
    _config_parity(sk, "c2")


def test_config_c3_full(sk):
    _config_parity(sk, "c3")


def test_config_c4_full(sk):
    _config_parity(sk, "c4")


def test_config_c5_full(sk):
    _config_parity(sk, "c5")


# ------------------------------------------------------------------- SAP least squares (§8(f) f2)

@pytest.mark.parametrize("dist,method", [("gaussian", "qr"), ("rademacher", "qr"), ("uniform", "svd")])
def test_sap_solve_on_gpu(sk, dist, method):
    # sketch-and-precondition LSQR with the fused kernel's Â on the GPU: the
    # paper's 1e-14 stopping rule is met in a few dozen iterations and x is the least-squares solution
    import torch
    from paper_2310_15419_b200 import sap
    A, b = workloads.ls_problem(60000, 150, 80, seed=41, col_scale_decades=2.0)
    res = sap.sap_solve(_dev(A.colptr), _dev(A.rowidx), _dev(A.vals), A.m, A.n, _dev(b), d=2 * A.n, seed=3,
                        dist=dist, method=method)
    assert res.istop in (1, 2) and res.iterations <= 80, (res.istop, res.iterations)
    assert res.error <= 1e-13, res.error
    M = np.zeros((A.m, A.n))
    for k in range(A.n):
        r, v = A.column(k)
        M[r, k] += v
    xref = np.linalg.lstsq(M, b, rcond=None)[0]
    x = res.x.cpu().numpy()
    assert np.linalg.norm(x - xref) <= 1e-8 * np.linalg.norm(xref)


# ------------------------------------------------------------------- Algorithm 4 (jki, §8(f) f1)

JKI_CASES = [
    ("abnormal_A", lambda: workloads.abnormal_paper("A", m=20000, n=70, seed=1), 700),
    ("abnormal_B", lambda: workloads.abnormal_paper("B", m=9000, n=60, seed=2), 300),
    ("abnormal_C", lambda: workloads.abnormal_paper("C", m=3000, n=2100, seed=3), 129),
    ("random_ragged", lambda: workloads.random_csc(5000, 37, [0, 3, 40, 1, 0, 200] * 6 + [7], seed=4), 1100),
    ("unsorted_dups", lambda: workloads.random_csc(300, 21, 60, seed=5, sorted_rows=False, duplicates=True), 65),
]


@pytest.mark.parametrize("dist", ["uniform", "gaussian"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("case", JKI_CASES, ids=[c[0] for c in JKI_CASES])
def test_jki_matches_oracle(sk, dist, dtype, case):
    # Algorithm 4 (one S[:, j] per nonzero row of a column block, reused across the row) gives the
    # same sketch as the oracle's Algorithm 3 loop, within the dtype's bar
    import torch
    name, build, d = case
    A = build()
    if dtype == "f32":
        A.vals = A.vals.astype(np.float32)
    plan = sk.Plan(_dev(A.colptr), _dev(A.rowidx), d, A.m, dtype, jki=True)
    try:
        sk.set_pair_path("jki")
        st = plan.stats()
        assert st["n_items_jki"] > 0 and "Algorithm 4" in plan.kernel_name(dist)
        got = plan.apply(_dev(A.vals), 19, dist).T.double().cpu().numpy()
        torch.cuda.synchronize()
    finally:
        sk.set_pair_path("auto")
        plan.close()
    ref, B = oracle.sketch(19, dist, d, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=8)
    _check(got, ref, B, TOL[dtype])


def test_jki_auto_selection(sk):
    # the plan builds the Algorithm 4 structure on its own only when the exact distinct-row count of
    # its column blocks (b_n = 384 fp64 columns) clears the loosest bar (f64 Gaussian: rows <= 0.40
    # nnz), and then uses it per distribution from the measured costs (sketch_api.cu):
    # rows/nnz = 0.016 (Abnormal A-like) -> Algorithm 4 for uniform and Gaussian S; 0.25 -> Gaussian
    # only (uniform needs <= 0.10); 0.95 -> not built
    A = workloads.abnormal_paper("A", m=20000, n=64, seed=1)
    M = workloads.random_csc(4900, 64, 300, seed=6)
    B = workloads.random_csc(200000, 64, 300, seed=2)
    pa = sk.Plan(_dev(A.colptr), _dev(A.rowidx), 256, A.m)
    pm = sk.Plan(_dev(M.colptr), _dev(M.rowidx), 256, M.m)
    pb = sk.Plan(_dev(B.colptr), _dev(B.rowidx), 256, B.m)
    try:
        assert pa.stats()["n_items_jki"] > 0 and pm.stats()["n_items_jki"] > 0 and pb.stats()["n_items_jki"] == 0
        # the RNG work of Algorithm 4 is exactly the distinct rows of every column block
        # (PAPER.md:302-318, 436-442): here one block of all 64 columns
        assert pa.stats()["jki_nonzero_rows"] == len(np.unique(A.rowidx))
        assert pm.stats()["jki_nonzero_rows"] == len(np.unique(M.rowidx))
        assert 0.10 < pm.stats()["jki_nonzero_rows"] / M.nnz <= 0.40
        assert "Algorithm 4" in pa.kernel_name("gaussian") and "Algorithm 4" in pa.kernel_name("uniform")
        assert "Algorithm 4" in pm.kernel_name("gaussian") and "Algorithm 4" not in pm.kernel_name("uniform")
        sk.set_pair_path("jki")
        assert "Algorithm 4" in pm.kernel_name("uniform")
        sk.set_pair_path("kji")
        assert "Algorithm 4" not in pa.kernel_name("gaussian")
    finally:
        sk.set_pair_path("auto")
        pa.close()
        pm.close()
        pb.close()


def test_jki_on_c2_with_exact_row_count(sk):
    # BASELINE config c2 (1000 distinct uniform rows per column of 1e6): a forced Algorithm 4 plan
    # generates every needed S column exactly once per column block -- its row count is exactly the
    # sum over the b_n-column blocks of their distinct rows -- and matches the oracle; the automatic
    # plan keeps Algorithm 3 (reuse too low)
    import torch
    A = workloads.make_config("c2")
    auto = sk.Plan(_dev(A.colptr), _dev(A.rowidx), 2000, A.m)
    assert auto.stats()["n_items_jki"] == 0
    auto.close()
    plan = sk.Plan(_dev(A.colptr), _dev(A.rowidx), 2000, A.m, jki=True)
    try:
        sk.set_pair_path("jki")
        st = plan.stats()
        bn = st["jki_block_cols"]
        assert bn > 0 and st["n_items_jki"] > 0
        want = sum(len(np.unique(A.rowidx[A.colptr[c]:A.colptr[min(c + bn, A.n)]])) for c in range(0, A.n, bn))
        assert st["jki_nonzero_rows"] == want
        got = plan.apply(_dev(A.vals), 1, "uniform").T.cpu().numpy()
        torch.cuda.synchronize()
    finally:
        sk.set_pair_path("auto")
        plan.close()
    cols = [0, 1, 499, 998, 999]
    As = A.select_columns(cols)
    ref, B = oracle.sketch(1, "uniform", 2000, As.m, As.n, As.colptr, As.rowidx, As.vals, threads=8)
    _check(got[:, cols], ref, B, TOL["f64"])


def test_jki_multiple_blocks_and_split_parts(sk):
    # n > b_n: several column blocks (Abnormal A-like dense rows so every block reuses its rows), a
    # row with more entries than one batch holds (duplicated entries in a dense row), and few row
    # tiles (d = 40) so each block's batches are split over several items and summed by the finishing
    # kernel; fp64 and fp32, uniform and Gaussian
    import torch
    rng = np.random.default_rng(3)
    m, n = 3000, 2300
    dense_rows = np.arange(0, m, 100)
    cols = []
    for k in range(n):
        r = np.concatenate([dense_rows, rng.choice(m, 3, replace=False)])
        if k % 2 == 0:
            r = np.concatenate([r, [7, 7, 7]])         # duplicate (j, k) entries, unsorted: row 7 holds
                                                       # > 512 entries (one batch) in every full block
        cols.append(r.astype(np.int32))
    colptr = np.zeros(n + 1, np.int64)
    colptr[1:] = np.cumsum([len(c) for c in cols])
    rowidx = np.concatenate(cols).astype(np.int32)
    vals = rng.standard_normal(int(colptr[-1]))
    for dtype in ("f64", "f32"):
        A = workloads.CSC(m, n, colptr, rowidx, vals.astype(np.float32 if dtype == "f32" else np.float64))
        for dist, d in (("uniform", 40), ("gaussian", 300)):
            plan = sk.Plan(_dev(A.colptr), _dev(A.rowidx), d, A.m, dtype)
            try:
                sk.set_pair_path("jki")
                assert plan.stats()["n_items_jki"] > 0 and "Algorithm 4" in plan.kernel_name(dist), dtype
                got = plan.apply(_dev(A.vals), 23, dist).T.double().cpu().numpy()
                got2 = plan.apply(_dev(A.vals), 23, dist).T.double().cpu().numpy()
                torch.cuda.synchronize()
            finally:
                sk.set_pair_path("auto")
                plan.close()
            assert np.array_equal(got, got2)
            ref, B = oracle.sketch(23, dist, d, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=8)
            _check(got, ref, B, TOL[dtype])
