"""Pins for the CPU oracle (tests run without a GPU).

Each test checks the oracle against something OTHER than itself (SURVEY.md §8(c) c.6,
DESIGN.md §"Oracle pins"):
  * Philox4x32-10 words  -> Triton's independent `tl.philox` run by its CPU interpreter,
                            plus bit-balance / avalanche statistics;
  * S entries           -> distribution laws (moments, KS tests), exact value-set
                            properties, prefix/blocking invariance, mpmath accuracy;
  * Â = S·A             -> brute-force dense numpy products, exact integer arithmetic,
                            A = I and single-nonzero special cases, linearity,
                            row-shard additivity, E[ÂᵀÂ]/(dσ²) = AᵀA, and the paper's
                            conditioning claim cond(A R⁻¹) ≲ 10 at d = 2n.
"""
import json
import os
import subprocess
import sys
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workloads

HERE = os.path.dirname(os.path.abspath(__file__))


# ------------------------------------------------------------------------- Philox words

def _triton_philox(cases):
    p = subprocess.run([sys.executable, os.path.join(HERE, "_triton_philox_ref.py")],
                       input=json.dumps(cases), capture_output=True, text=True, timeout=600)
    if p.returncode != 0:
        pytest.skip(f"triton interpreter unavailable: {p.stderr[-300:]}")
    return json.loads(p.stdout)


def test_philox_matches_independent_triton_implementation():
    rng = np.random.default_rng(123)
    cases = [[0, 0, 0, 0, 0, 0], [0xFFFFFFFF] * 6]
    for _ in range(200):
        cases.append([int(x) for x in rng.integers(0, 2**32, size=6, dtype=np.uint64)])
    # counters in the layout the sketch uses: (q, 0, j_lo, j_hi), key = seed halves
    for q, j, seed in [(0, 0, 0), (1, 0, 0), (0, 1, 0), (15, 49_999_999, 4), (127, 2**32 + 5, 2**40 + 3)]:
        cases.append([q, 0, j & 0xFFFFFFFF, j >> 32, seed & 0xFFFFFFFF, seed >> 32])
    ref = _triton_philox(cases)
    for c, r in zip(cases, ref):
        assert oracle.philox4x32_10(c[:4], c[4:]) == tuple(r), c


def test_philox_bit_balance_and_avalanche():
    # every output bit is a fair coin over many counters (binomial 5-sigma window)
    N = 20000
    counts = np.zeros(128)
    for q in range(N):
        x = oracle.philox4x32_10([q, 0, 12345, 0], [99, 0])
        bits = np.unpackbits(np.array(x, dtype="<u4").view(np.uint8), bitorder="little")
        counts += bits
    p = counts / N
    assert np.all(np.abs(p - 0.5) < 5 * 0.5 / np.sqrt(N))
    # avalanche: flipping one counter bit flips ~half of the 128 output bits
    flips = []
    for t in range(200):
        c = [t, 7, 3, 1]
        x0 = np.array(oracle.philox4x32_10(c, [1, 2]), dtype=np.uint32)
        c2 = list(c)
        c2[t % 4] ^= 1 << (t % 32)
        x1 = np.array(oracle.philox4x32_10(c2, [1, 2]), dtype=np.uint32)
        flips.append(np.unpackbits((x0 ^ x1).view(np.uint8)).sum())
    assert 60 < np.mean(flips) < 68


# ------------------------------------------------------------------------- S entries

@pytest.mark.parametrize("dist", ["rademacher", "uniform", "gaussian", "uniform24"])
def test_entrywise_equals_blockwise_generation(dist):
    # S[i, j] must not depend on how it is generated (block reuse vs one entry at a time)
    # nor on d (prefix property, R16): the reproducibility the paper asks of a
    # CBRNG.
    for j in [0, 1, 77, 2**31 + 3]:
        v = oracle.get_samples(11, dist, j, 300)
        w = np.array([oracle.s_entry(11, dist, i, j) for i in range(300)])
        assert np.array_equal(v, w)
        assert np.array_equal(oracle.get_samples(11, dist, j, 131), v[:131])


def test_rademacher_law():
    S = oracle.fill_s(5, "rademacher", 0, 512, 0, 400)
    assert set(np.unique(S)) == {-1.0, 1.0}
    N = S.size
    assert abs(S.mean()) < 5 / np.sqrt(N)
    # rows and columns are uncorrelated: sample correlation between two columns ~ 0
    c = (S[:, :200] * S[:, 200:]).mean()
    assert abs(c) < 5 / np.sqrt(S[:, :200].size)


def test_uniform_law_and_exact_grid():
    from scipy import stats
    S = oracle.fill_s(6, "uniform", 0, 400, 0, 300).ravel()
    assert np.all(np.abs(S) < 1.0)                        # open interval (-1, 1)
    odd = S * 2.0**53                                     # exact: values live on the odd grid
    assert np.all(odd == np.round(odd)) and np.all(np.mod(odd, 2) == 1)
    N = S.size
    assert abs(S.mean()) < 5 * np.sqrt(1 / 3 / N)
    assert abs((S**2).mean() - 1 / 3) < 5 * np.sqrt(4 / 45 / N)   # Var U(-1,1) = 1/3
    assert stats.kstest(S, stats.uniform(loc=-1, scale=2).cdf).pvalue > 1e-4


def test_uniform_word_order_against_independent_philox():
    # SK_UNIFORM's entry 2q + h is built from words (x[2h], x[2h+1]) of block q as U = x[2h] 2^32 +
    # x[2h+1], k = U >> 11, S = (2k + 1 - 2^53) 2^-53 (R2).  Pinned to Triton's independent
    # Philox words, so a swapped word order (x[2h+1] 2^32 + x[2h]) or a wrong shift fails here, not
    # only on the GPU; the ±1 bit order (entry 128q + 32t + b = bit b of word t, R3) likewise.
    seed, j = 2**35 + 77, 2**32 + 3
    words = _triton_philox([[q, 0, j & 0xFFFFFFFF, j >> 32, seed & 0xFFFFFFFF, seed >> 32] for q in range(4)])
    col = oracle.get_samples(seed, "uniform", j, 8)
    for q in range(4):
        for h in range(2):
            U = (int(words[q][2 * h]) << 32) | int(words[q][2 * h + 1])
            k = U >> 11
            assert col[2 * q + h] == (2 * k + 1 - 2**53) / 2.0**53
    rad = oracle.get_samples(seed, "rademacher", j, 512)
    for q in range(4):
        for t in range(4):
            for b in range(32):
                bit = (int(words[q][t]) >> b) & 1
                assert rad[128 * q + 32 * t + b] == (-1.0 if bit else 1.0)


def test_uniform24_law_exact_grid_and_words():
    # the 24-bit odd grid, 4 entries per Philox block.  Pinned to the law (open
    # interval, exact grid, mean 0, variance (1 - 2^-48)/3, KS) and to the Philox words through the
    # independent Triton reference: entry 4q + t uses the top 24 bits of word t of block q.
    from scipy import stats
    S = oracle.fill_s(16, "uniform24", 0, 400, 0, 300).ravel()
    assert np.all(np.abs(S) < 1.0)
    odd = S * 2.0**24
    assert np.all(odd == np.round(odd)) and np.all(np.mod(odd, 2) == 1)
    assert np.array_equal(S.astype(np.float32).astype(np.float64), S)   # exact in fp32
    N = S.size
    assert abs(S.mean()) < 5 * np.sqrt(1 / 3 / N)
    assert abs((S**2).mean() - 1 / 3) < 5 * np.sqrt(4 / 45 / N)
    assert stats.kstest(S, stats.uniform(loc=-1, scale=2).cdf).pvalue > 1e-4
    seed, j = 2**40 + 9, 5
    words = _triton_philox([[q, 0, j, 0, seed & 0xFFFFFFFF, seed >> 32] for q in range(3)])
    col = oracle.get_samples(seed, "uniform24", j, 12)
    for q in range(3):
        for t in range(4):
            k = int(words[q][t]) >> 8
            assert col[4 * q + t] == (2 * k + 1 - 2**24) / 2.0**24


def test_gaussian_law():
    from scipy import stats
    S = oracle.fill_s(7, "gaussian", 0, 400, 0, 300).ravel()
    N = S.size
    assert abs(S.mean()) < 5 / np.sqrt(N)
    assert abs((S**2).mean() - 1) < 5 * np.sqrt(2 / N)
    assert abs((S**4).mean() - 3) < 5 * np.sqrt(96 / N)
    assert stats.kstest(S, "norm").pvalue > 1e-4
    # the Box-Muller pair (S[2q], S[2q+1]) is rotation invariant: angle uniform on (-pi, pi]
    ang = np.arctan2(S.reshape(-1, 2)[:, 1], S.reshape(-1, 2)[:, 0])
    assert stats.kstest(ang, stats.uniform(loc=-np.pi, scale=2 * np.pi).cdf).pvalue > 1e-4


def test_gaussian_libm_accuracy_vs_mpmath():
    # Accuracy of the oracle's libm log/sqrt/cos/sin against 50-digit arithmetic on the
    # same Philox words: this bounds the oracle's own error well below the 1e-14 parity bar.
    import mpmath
    mpmath.mp.dps = 50
    for j in range(20):
        for q in range(10):
            x = oracle.philox4x32_10([q, 0, j, 0], [9, 0])
            k1 = ((x[0] << 32) | x[1]) >> 11
            k2 = ((x[2] << 32) | x[3]) >> 11
            u1 = mpmath.mpf(k1 + 1) / 2**53
            th = mpmath.mpf(float(np.float64(k2 * 2.0**-53) * np.float64(6.283185307179586)))
            rho = mpmath.sqrt(-2 * mpmath.log(u1))
            for e, f in ((0, mpmath.cos), (1, mpmath.sin)):
                exact = rho * f(th)
                got = oracle.s_entry(9, "gaussian", 2 * q + e, j)
                assert abs(got - float(exact)) <= 4e-16 * abs(float(exact)) + 1e-300


def test_f32_entries_are_rn_even_of_f64():
    for dist in ("uniform", "gaussian"):
        S64 = oracle.fill_s(3, dist, 0, 64, 0, 64)
        S32 = oracle.fill_s(3, dist, 0, 64, 0, 64, dtype="f32")
        assert np.array_equal(S32, S64.astype(np.float32).astype(np.float64))


# ------------------------------------------------------------------------- Â = S·A

def _dense_check(A, dist, d, seed, dtype="f64"):
    Ahat, B = oracle.sketch(seed, dist, d, A.m, A.n, A.colptr, A.rowidx, A.vals,
                            row_offset=A.row_offset)
    S = oracle.fill_s(seed, dist, 0, d, A.row_offset, A.row_offset + A.m,
                      dtype=("f32" if A.vals.dtype == np.float32 else "f64"))
    Ad = A.to_dense()
    ref = S @ Ad
    bnd = np.abs(S) @ np.abs(Ad)
    return Ahat, B, ref, bnd


@pytest.mark.parametrize("dist", ["rademacher", "uniform", "gaussian", "uniform24"])
def test_sketch_matches_bruteforce_dense_product(dist):
    A = workloads.random_csc(300, 12, 9, seed=1)
    Ahat, B, ref, bnd = _dense_check(A, dist, 70, seed=42)
    assert np.allclose(B, bnd, rtol=1e-13, atol=0)
    assert np.all(np.abs(Ahat - ref) <= 1e-13 * bnd)


def test_sketch_exact_for_rademacher_smallint():
    # ±1 S with small-integer A: every partial sum is an exact integer, so Â must equal the
    # exact rational product computed with Python integers.
    A = workloads.random_csc(200, 6, 15, seed=2, values="smallint")
    d = 50
    Ahat, _ = oracle.sketch(3, "rademacher", d, A.m, A.n, A.colptr, A.rowidx, A.vals)
    S = oracle.fill_s(3, "rademacher", 0, d, 0, A.m)
    for k in range(A.n):
        r, v = A.column(k)
        for i in range(d):
            exact = sum(Fraction(int(S[i, int(j)])) * Fraction(int(a)) for j, a in zip(r, v))
            assert Ahat[i, k] == float(exact)


@pytest.mark.parametrize("dist", ["rademacher", "uniform", "gaussian"])
def test_identity_gives_S_and_single_nonzero(dist):
    m = 40
    A = workloads.CSC(m, m, np.arange(m + 1, dtype=np.int64), np.arange(m, dtype=np.int32),
                      np.ones(m))
    Ahat, _ = oracle.sketch(8, dist, 33, m, m, A.colptr, A.rowidx, A.vals)
    assert np.array_equal(Ahat, oracle.fill_s(8, dist, 0, 33, 0, m))        # A = I => Â = S
    # one nonzero a at (j, k): column k is a * S[:, j] (one rounded product), others 0
    a, j = -2.5, 17
    colptr = np.array([0, 0, 1, 1], dtype=np.int64)
    Ahat, _ = oracle.sketch(8, dist, 33, m, 3, colptr, np.array([j], np.int32), np.array([a]))
    assert np.array_equal(Ahat[:, 1], a * oracle.fill_s(8, dist, 0, 33, j, j + 1)[:, 0])
    assert not Ahat[:, [0, 2]].any()


def test_linearity_in_A():
    A1 = workloads.random_csc(500, 8, 12, seed=4)
    A2 = workloads.random_csc(500, 8, 12, seed=5)
    alpha = 0.75
    S1, _ = oracle.sketch(1, "uniform", 64, 500, 8, A1.colptr, A1.rowidx, A1.vals)
    S2, _ = oracle.sketch(1, "uniform", 64, 500, 8, A2.colptr, A2.rowidx, A2.vals)
    # αA1 + A2 as a CSC with duplicate (j, k) entries (accepted by linearity, reading R9)
    colptr = A1.colptr + A2.colptr
    rows, vals = [], []
    for k in range(8):
        r1, v1 = A1.column(k)
        r2, v2 = A2.column(k)
        rows.append(np.concatenate([r1, r2]))
        vals.append(np.concatenate([alpha * v1, v2]))
    S12, B = oracle.sketch(1, "uniform", 64, 500, 8, colptr, np.concatenate(rows).astype(np.int32),
                           np.concatenate(vals))
    assert np.all(np.abs(S12 - (alpha * S1 + S2)) <= 1e-14 * (B + 1e-300))


def test_row_shards_add_up():
    # Row sharding: Σ_g sketch(A_g, row_offset = r_g) = sketch(A)
    A = workloads.random_csc(1000, 10, 30, seed=6)
    full, B = oracle.sketch(2, "rademacher", 100, A.m, A.n, A.colptr, A.rowidx, A.vals)
    tot = np.zeros_like(full)
    for g in range(3):
        Ag = workloads.shard_csc(A, 3, g)
        part, _ = oracle.sketch(2, "rademacher", 100, Ag.m, Ag.n, Ag.colptr, Ag.rowidx, Ag.vals,
                                row_offset=Ag.row_offset)
        tot += part
    assert np.all(np.abs(tot - full) <= 1e-14 * B)


def test_threads_do_not_change_result():
    A = workloads.random_csc(2000, 40, 25, seed=7)
    a1, _ = oracle.sketch(3, "gaussian", 90, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=1)
    a4, _ = oracle.sketch(3, "gaussian", 90, A.m, A.n, A.colptr, A.rowidx, A.vals, threads=4)
    assert np.array_equal(a1, a4)


@pytest.mark.parametrize("dist,sigma2", [("rademacher", 1.0), ("uniform", 1 / 3), ("gaussian", 1.0),
                                          ("uniform24", 1 / 3)])
def test_expected_gram_matches_AtA(dist, sigma2):
    # North-star invariant: E[ÂᵀÂ] / (d σ²) = AᵀA (R15), averaged over seeds.
    A = workloads.random_csc(60, 4, 6, seed=8)
    Ad = A.to_dense()
    G = Ad.T @ Ad
    d, nseeds = 16, 600
    acc = np.zeros_like(G)
    sq = np.zeros_like(G)
    for s in range(nseeds):
        Ah, _ = oracle.sketch(1000 + s, dist, d, A.m, A.n, A.colptr, A.rowidx, A.vals,
                              want_bound=False)
        g = Ah.T @ Ah / (d * sigma2)
        acc += g
        sq += g * g
    mean = acc / nseeds
    se = np.sqrt(np.maximum(sq / nseeds - mean**2, 1e-30) / nseeds)
    assert np.all(np.abs(mean - G) <= 5 * se + 1e-12)


def test_sketch_preconditions_tall_matrix():
    # with d = γn the sketch gives cond(A R⁻¹) ≤ (√γ+1)/(√γ−1) (Gaussian,
    # asymptotically); the draft checks cond ≲ 10 at d = 2n.
    A = workloads.random_csc(3000, 40, 60, seed=9)
    Ad = A.to_dense()
    for dist in ("rademacher", "uniform", "gaussian"):
        Ah, _ = oracle.sketch(17, dist, 80, A.m, A.n, A.colptr, A.rowidx, A.vals, want_bound=False)
        R = np.linalg.qr(Ah, mode="r")
        c = np.linalg.cond(Ad @ np.linalg.inv(R))
        assert c < 10, (dist, c)


def test_edge_cases_empty_and_zero():
    # n = 0, nnz = 0, empty columns, explicit zeros
    out, B = oracle.sketch(1, "rademacher", 5, 10, 0, np.zeros(1, np.int64), np.zeros(0, np.int32),
                           np.zeros(0))
    assert out.shape == (5, 0)
    colptr = np.array([0, 0, 2, 2], np.int64)
    out, B = oracle.sketch(1, "uniform", 7, 10, 3, colptr, np.array([3, 4], np.int32),
                           np.array([0.0, 0.0]))
    assert not out.any() and not B.any()
    with pytest.raises(ValueError):
        oracle.sketch(1, "uniform", 7, 10, 1, np.array([0, 1], np.int64), np.array([10], np.int32),
                      np.array([1.0]))


def test_paper_gflops_metric_golden():
    # tests/golden/paper_tab_parallel.csv: Table tab:parallel prints both
    # time and GFlops for shar_te2-b2 (d, nnz from Table matrix:name);
    # the metric 2·d·nnz/t must reproduce every printed GFlops within print rounding.
    from paper_2310_15419_b200.metrics import gflops
    import csv
    path = os.path.join(HERE, "golden", "paper_tab_parallel.csv")
    rows = list(csv.DictReader(l for l in open(path) if not l.startswith("#")))
    assert len(rows) == 24
    for r in rows:
        t = float(r["time_s"])
        g = gflops(int(r["d"]), int(r["nnz"]), t)
        tol = g * (0.005 / t) + 0.006            # time printed to 0.01 s, GFlops to 0.01
        assert abs(g - float(r["gflops"])) <= tol, r


def test_expected_nonzero_rows_formula():
    # PAPER.md:361-365 (cost model): with entries nonzero independently with probability rho,
    # the number Y of rows of an m1 x n1 block holding a nonzero has E[Y] = m1 (1 - (1-rho)^n1).
    # Pinned by simulation (not by retyping the formula): mean of Y over many Bernoulli blocks,
    # within 5 standard errors, for several (m1, n1, rho); and the limits rho = 0, rho = 1, n1 = 1.
    from paper_2310_15419_b200.metrics import expected_nonzero_rows
    rng = np.random.default_rng(365)
    for m1, n1, rho in ((1000, 16, 0.01), (500, 4, 0.2), (2000, 64, 0.002)):
        trials = 400
        ys = np.array([(rng.random((m1, n1)) < rho).any(axis=1).sum() for _ in range(trials)], dtype=float)
        se = ys.std(ddof=1) / np.sqrt(trials)
        assert abs(ys.mean() - expected_nonzero_rows(m1, n1, rho)) <= 5 * se + 1e-9, (m1, n1, rho)
    assert expected_nonzero_rows(100, 8, 0.0) == 0.0
    assert expected_nonzero_rows(100, 8, 1.0) == 100.0
    assert abs(expected_nonzero_rows(100, 1, 0.3) - 30.0) < 1e-12
