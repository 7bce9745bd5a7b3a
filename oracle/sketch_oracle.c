/*
 * sketch_oracle.c -- plain, slow, obviously-correct CPU oracle for the sketch  Â = S·A
 * of arXiv 2310.15419 ("blocking and on-the-fly RNG for sketching sparse matrices").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this file.  The product path
 * (paper_2310_15419_b200/, libsketch.so) shares NO code, header, table or constant
 * generator with it; the two are independent implementations of the definitions
 * below, and agreement between them is the parity evidence.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 *        (no contraction, so every product/sum below is one IEEE fp64 operation).
 *
 * What it computes (everything in fp64, indices 0-based -- DESIGN.md reading R10):
 *
 *  (1) Philox4x32-10 (the "counter based RNG ... Random123" of PAPER.md:489-492,
 *      §4.2 "Counter Based RNG"; the paper says to "use the row-column indices of the
 *      elements in the matrices as counters").  Written out from the
 *      Salmon et al. round definition; no blocking, no vectorisation.
 *      Counter layout (reading R1): entry S[i, j] lives in the block
 *      ctr = (q, 0, j mod 2^32, j div 2^32), key = (seed mod 2^32, seed div 2^32).
 *
 *  (2) The entry distributions of PAPER.md:30 ("mean-zero Gaussian, uniform over
 *      (-1, 1), or simply uniform over ±1") via the transforms of DESIGN.md R2-R4:
 *        Rademacher  q = i/128, word t = (i%128)/32, bit b = i%32; bit=1 -> -1 else +1
 *        Uniform     q = i/2, h = i%2, U = x[2h]*2^32 + x[2h+1], k = U>>11,
 *                    S = (2k + 1 - 2^53) * 2^-53          (exact odd grid in (-1,1))
 *        Gaussian    q = i/2, k1 = U1>>11, k2 = U2>>11, u1 = (k1+1)2^-53, u2 = k2 2^-53,
 *                    rho = sqrt(-2 ln u1), th = u2 * fl(2 pi),
 *                    S[2q] = rho cos th, S[2q+1] = rho sin th   (Box-Muller)
 *        Uniform24   (the 32-bit numbers of PAPER.md:464): a cheaper
 *                    uniform(-1, 1) with 4 entries per block: q = i/4, t = i%4,
 *                    k = x[t] >> 8 (24 bits), S = (2k + 1 - 2^24) * 2^-24 (odd grid, exact in
 *                    fp32 and fp64)
 *      For dtype F32 the entry is RN-even(S64) (R5).
 *
 *  (3) The sketch itself in the loop order of Algorithm 3 "Variant kji with RNG"
 *      (PAPER.md:259-286): for every column k, for every stored nonzero (j, a) of
 *      column k in storage order, regenerate v = S[:, j] (PAPER.md:275-276,
 *      "g.set_state(r, j); g.get_samples(v)") and do  Â[:, k] += a * v
 *      (PAPER.md:277-278).  Â starts at 0 (Algorithm 1).  It also returns
 *      the error-bound matrix B = |S|·|A| used by the parity tolerance.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

enum { OR_RADEMACHER = 0, OR_UNIFORM = 1, OR_GAUSSIAN = 2, OR_UNIFORM24 = 3 };
enum { OR_F64 = 0, OR_F32 = 1 };

/* ---------------------------------------------------------------------------------
 * Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), the Random123 generator the paper
 * names at PAPER.md:490.  One round:
 *     (hi0, lo0) = M0 * c0,   (hi1, lo1) = M1 * c2          (32x32 -> 64-bit products)
 *     c' = (hi1 ^ c1 ^ k0,  lo1,  hi0 ^ c3 ^ k1,  lo0)
 * ten rounds, the key bumped by the Weyl constants between rounds.
 * ------------------------------------------------------------------------------- */
void or_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    int round;
    for (round = 0; round < 10; ++round) {
        uint64_t p0 = (uint64_t)M0 * (uint64_t)c0;
        uint64_t p1 = (uint64_t)M1 * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += W0;  /* key schedule: bump after every round (the bump after round 10 is unused) */
        k1 += W1;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* The Philox block holding entry S[i, j]: counter (q, 0, j_lo, j_hi), key = seed halves. */
static void block_for(uint64_t seed, uint64_t q, uint64_t j, uint32_t x[4])
{
    uint32_t ctr[4], key[2];
    ctr[0] = (uint32_t)q;
    ctr[1] = (uint32_t)(q >> 32);
    ctr[2] = (uint32_t)j;
    ctr[3] = (uint32_t)(j >> 32);
    key[0] = (uint32_t)seed;
    key[1] = (uint32_t)(seed >> 32);
    or_philox4x32_10(ctr, key, x);
}

/* 2*pi rounded to the nearest double (0x1.921fb54442d18p+2), reading R4. */
static const double OR_TWO_PI = 6.283185307179586231995926937088;

/* Entry e of Philox block x (e in [0, E)), in fp64, straight from the definitions above. */
static double entry_from_block(int dist, const uint32_t x[4], int e)
{
    if (dist == OR_RADEMACHER) {           /* E = 128: word t = e/32, bit b = e%32 */
        int t = e / 32, b = e % 32;
        return ((x[t] >> b) & 1u) ? -1.0 : 1.0;
    } else if (dist == OR_UNIFORM) {       /* E = 2: entry h uses words (2h, 2h+1) */
        int h = e;
        uint64_t U = ((uint64_t)x[2 * h] << 32) | (uint64_t)x[2 * h + 1];
        uint64_t k = U >> 11;                                     /* 53 random bits */
        int64_t odd = (int64_t)(2u * k + 1u) - ((int64_t)1 << 53); /* odd, |odd| < 2^53: exact */
        return (double)odd * 0x1p-53;
    } else if (dist == OR_UNIFORM24) {     /* E = 4: entry t uses the top 24 bits of word t */
        uint32_t k = x[e] >> 8;
        int32_t odd = (int32_t)(2u * k + 1u) - (int32_t)(1 << 24);   /* odd, |odd| < 2^24: exact */
        return (double)odd * 0x1p-24;
    } else {                               /* E = 2: Box-Muller pair */
        uint64_t U1 = ((uint64_t)x[0] << 32) | (uint64_t)x[1];
        uint64_t U2 = ((uint64_t)x[2] << 32) | (uint64_t)x[3];
        uint64_t k1 = U1 >> 11, k2 = U2 >> 11;
        double u1 = (double)(k1 + 1u) * 0x1p-53;   /* (0, 1] : ln never sees 0 */
        double u2 = (double)k2 * 0x1p-53;          /* [0, 1) */
        double rho = sqrt(-2.0 * log(u1));
        double th = u2 * OR_TWO_PI;
        return (e == 0) ? rho * cos(th) : rho * sin(th);
    }
}

static int entries_per_block(int dist) { return dist == OR_RADEMACHER ? 128 : (dist == OR_UNIFORM24 ? 4 : 2); }

static double to_dtype(double v, int dtype)
{
    if (dtype == OR_F32) {
        float f = (float)v;   /* C conversion under the default rounding mode: RN-even */
        return (double)f;
    }
    return v;
}

/* One entry S[i, j] (definition applied to a single index; no reuse between entries). */
double or_s_entry_f64(uint64_t seed, int dist, int64_t i, int64_t j)
{
    uint32_t x[4];
    int E = entries_per_block(dist);
    block_for(seed, (uint64_t)i / (uint64_t)E, (uint64_t)j, x);
    return entry_from_block(dist, x, (int)((uint64_t)i % (uint64_t)E));
}

/* get_samples of Algorithm 3: v[0..d) = S[0..d, j],
 * generated block by block in increasing q (entries past d in the last block dropped). */
void or_get_samples(uint64_t seed, int dist, int dtype, int64_t j, int64_t d, double* v)
{
    uint32_t x[4];
    int E = entries_per_block(dist);
    int64_t q, nq = (d + E - 1) / E;
    for (q = 0; q < nq; ++q) {
        int e;
        block_for(seed, (uint64_t)q, (uint64_t)j, x);
        for (e = 0; e < E; ++e) {
            int64_t i = q * E + e;
            if (i < d) v[i] = to_dtype(entry_from_block(dist, x, e), dtype);
        }
    }
}

/* Entry in the requested storage dtype, returned widened to double (exactly). */
double or_s_entry(uint64_t seed, int dist, int dtype, int64_t i, int64_t j)
{
    return to_dtype(or_s_entry_f64(seed, dist, i, j), dtype);
}

/* Materialise S[i0:i1, j0:j1] column-major ((i1-i0) x (j1-j0)), one entry at a time. */
int or_fill_s(uint64_t seed, int dist, int dtype, int64_t i0, int64_t i1, int64_t j0, int64_t j1,
              double* out)
{
    int64_t i, j, rows = i1 - i0;
    if (i1 < i0 || j1 < j0 || i0 < 0 || j0 < 0 || dist < 0 || dist > 3 || dtype < 0 || dtype > 1)
        return -1;
    for (j = j0; j < j1; ++j)
        for (i = i0; i < i1; ++i)
            out[(j - j0) * rows + (i - i0)] = or_s_entry(seed, dist, dtype, i, j);
    return 0;
}

/*
 * Â = S[:, row_offset : row_offset+m] · A   (A is m x n CSC, 0-based, int64 colptr,
 * int32 rowidx; vals given as fp64 -- fp32 inputs are widened exactly by the caller).
 * out, bound: d x n column-major fp64 (ld = d), overwritten.
 * Algorithm 3 (kji) order; nthreads > 1 splits the k loop only (each column keeps its
 * own summation order, so the result is bit-identical to nthreads = 1).
 */
int or_sketch(uint64_t seed, int dist, int dtype, int64_t d, int64_t m, int64_t n,
              int64_t row_offset, const int64_t* colptr, const int32_t* rowidx,
              const double* vals, double* out, double* bound, int nthreads)
{
    int64_t k;
    int bad = 0;
    if (d < 1 || m < 0 || n < 0 || row_offset < 0) return -1;
    if (n > 0 && colptr[0] != 0) return -2;
    for (k = 0; k < n; ++k) {
        int64_t p;
        if (colptr[k + 1] < colptr[k]) return -2;
        for (p = colptr[k]; p < colptr[k + 1]; ++p)
            if (rowidx[p] < 0 || (int64_t)rowidx[p] >= m) return -2;
    }
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads) reduction(|| : bad)
#endif
    for (k = 0; k < n; ++k) {
        int64_t i, p;
        double* v = (double*)malloc((size_t)d * sizeof(double));
        double* col = out + k * d;
        double* bcol = bound ? bound + k * d : NULL;
        if (!v) { bad = 1; continue; }
        for (i = 0; i < d; ++i) col[i] = 0.0;                  /* Â = 0 */
        if (bcol) for (i = 0; i < d; ++i) bcol[i] = 0.0;
        for (p = colptr[k]; p < colptr[k + 1]; ++p) {
            int64_t j = row_offset + (int64_t)rowidx[p];
            double a = vals[p];
            or_get_samples(seed, dist, dtype, j, d, v);           /* set_state(r,j); get_samples(v) */
            for (i = 0; i < d; ++i) col[i] += a * v[i];        /* Â[i,k] += A[j,k] * v[i] */
            if (bcol) for (i = 0; i < d; ++i) bcol[i] += fabs(a) * fabs(v[i]);
        }
        free(v);
    }
    return bad ? -3 : 0;
}

/* Number of host threads OpenMP would use (reported as `cores` of the CPU baseline). */
int or_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
