// philox.cuh -- device-side Philox4x32-10 and the entry transforms of include/sketch.h.
//
// Product code for sm_100a.  Shares nothing with oracle/ (independent implementation of
// the same definitions; agreement is the parity evidence).
//
// Philox4x32-10 is the counter-based generator family the paper names for reproducible
// on-the-fly generation ("use the row-column indices of the elements in the matrices as
// counters", §4.2; RandBLAS policy PAPER.md:508-513).  The ten round
// keys are precomputed on the host and passed as kernel parameters, so on sm_100a each
// round is 2 IMAD.WIDE.U32 (the two 32x32->64 products) + 2 LOP3 (3-input XOR with a
// constant-bank key operand): 40 integer instructions per 128 random bits.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "bm_tables.h"

namespace sk {

constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

// Round keys (k0 + r*W0, k1 + r*W1) for r = 0..9; lives in the kernel parameter bank.
struct PhiloxKeys {
  uint32_t k0[10];
  uint32_t k1[10];
};

inline PhiloxKeys make_keys(uint64_t seed) {
  PhiloxKeys K;
  uint32_t a = (uint32_t)seed, b = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    K.k0[r] = a;
    K.k1[r] = b;
    a += kPhiloxW0;
    b += kPhiloxW1;
  }
  return K;
}

// One Philox4x32-10 block: counter (c0, c1, c2, c3) under the precomputed keys.
__device__ __forceinline__ uint4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                               const PhiloxKeys& K) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)kPhiloxM0 * (uint64_t)c0;   // IMAD.WIDE.U32
    const uint64_t p1 = (uint64_t)kPhiloxM1 * (uint64_t)c2;   // IMAD.WIDE.U32
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ K.k0[r];  // LOP3
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ K.k1[r];  // LOP3
    c1 = (uint32_t)p1;
    c3 = (uint32_t)p0;
    c0 = n0;
    c2 = n2;
  }
  return make_uint4(c0, c1, c2, c3);
}

// Block holding S[i, j]: counter (q, 0, j mod 2^32, j div 2^32).
__device__ __forceinline__ uint4 s_block(uint32_t q, uint64_t j, const PhiloxKeys& K) {
  return philox4x32_10(q, 0u, (uint32_t)j, (uint32_t)(j >> 32), K);
}

// ---------------------------------------------------------------- transforms

// Uniform (-1, 1) on the odd 2^-53 grid: k = (xa:xb) >> 11, S = (2k + 1 - 2^53) 2^-53.
// k < 2^53 converts to double exactly (I2F.F64.U64 on the conversion pipe, off the busy ALU
// pipe), and S = fma(k, 2^-52, -(1 - 2^-53)) is exact: the true value is an odd multiple of
// 2^-53 of magnitude < 1, so the single rounding of the FMA changes nothing.
__device__ __forceinline__ double uniform53(uint32_t xa, uint32_t xb) {
  const unsigned long long k = (((unsigned long long)xa << 32) | xb) >> 11;
  return fma(__ull2double_rn(k), 0x1p-52, __longlong_as_double((long long)0xBFEFFFFFFFFFFFFFull));
}

// Uniform24: S = (2k + 1 - 2^24) 2^-24 with k = the top 24 bits of one
// Philox word (4 entries per block).  An odd multiple of 2^-24 below 1 in magnitude: exact in fp32
// (and fp64); I2F of the exact odd integer and one exact scaling.
__device__ __forceinline__ float uniform24(uint32_t w) {
  const int odd = (int)(((w >> 8) << 1) | 1u) - (1 << 24);
  return __int2float_rn(odd) * 0x1p-24f;
}


// ---------------------------------------------------------------- Box-Muller (fast fp64)
//
// Box-Muller pair from one block (include/sketch.h, R4): u1 = (k1 + 1) 2^-53 in (0, 1],
// u2 = k2 2^-53 in [0, 1), rho = sqrt(-2 ln u1), th = u2 * fl(2 pi); (g0, g1) = (rho cos th, rho sin th),
// with the library's own log and sincos (scripts/gen_bm_tables.py derives and checks the constants
// against 300-bit mpmath: <= 0.6 ulp each; ~40 FP64 operations per pair).  Results agree with the
// libm-based oracle far inside the Gaussian parity bound (1e-14 relative).

// The -2 log table in shared memory: one copy in 32-byte rows {-2c, 2 L_hi, 2 L_lo, 0} (4.1 KB; STRIDE = 0
// below), or replicated (STRIDE copies, copy c of row i component t at [(3 i + t) STRIDE + c], lane l
// reading copy l mod STRIDE: a half-warp's loads of any row mix then hit distinct bank pairs).
constexpr int kLogTab4Bytes = kBmLogRows * 4 * 8;
__device__ __forceinline__ void bm_fill_logtab4(double* smem_tab) {
  for (int i = threadIdx.x; i < kBmLogRows * 4; i += blockDim.x)
    smem_tab[i] = (i & 3) == 3 ? 0.0 : kBmLogTab[i >> 2][i & 3];
}

// -2 log(u1) for u1 = U 2^-53, U = k1 + 1 an integer in [1, 2^53] passed as an exact double (so
// u1's scaling costs no multiply: exponent bias 53).  u = 2^e m, idx = round(128 (m - 1)), and with
// the table rows {-2 c, 2 log(c)_hi, 2 log(c)_lo}: s = fma(m, -2c, 2) = -2 (m c - 1) exactly
// (|s| < 0.009), -2 log u = (e (-2 ln2_hi) + 2 L_hi) + (s + s^2 Q(s) + (e (-2 ln2_lo) + 2 L_lo)),
// Q(s) = 1/4 + s/12 + s^2/32 + s^3/80 + s^4/192 (= -P(-s/2)/2 for the Taylor P of
// (log1p(r) - r) / r^2, truncated where the next term is below 2^-60), the first bracket exact
// (2^-42 grid).  The factor -2 of Box-Muller is folded into the constants: 11 FP64 operations.
// tab = row 0, component 0 of this lane's copy; STRIDE = distance between consecutive components
// (the replication of a replicated table, 1 for kBmLogTab itself), or STRIDE = 0: one copy in 32-byte
// rows (bm_fill_logtab4).
template <int STRIDE>
__device__ __forceinline__ double bm_m2log_u53(double U, const double* __restrict__ tab) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(U);
  const int e = (int)(b >> 52) - (1023 + 53);
  const double m = __longlong_as_double((long long)((b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull));
  const int idx = (int)(((b >> 44) & 0xFFu) + 1u) >> 1;        // round(128 (m - 1)), 0..128
  double c2, hi, lo;
  if constexpr (STRIDE == 0) {        // one copy with 32-byte rows {-2c, 2 L_hi, 2 L_lo, pad}: 16 + 8 byte loads
    const double2 ch = *reinterpret_cast<const double2*>(tab + 4 * idx);
    c2 = ch.x; hi = ch.y; lo = tab[4 * idx + 2];
  } else {
    const double* row = tab + 3 * STRIDE * idx;
    c2 = row[0]; hi = row[STRIDE]; lo = row[2 * STRIDE];
  }
  const double s = fma(m, c2, 2.0);                            // -2 r, |r| < 0.0045
  const double s2 = s * s;
  double q = fma(s, kBm[kQ4], kBm[kQ3]);                       // (the s^5/448 term is below 2^-60)
  q = fma(s, q, kBm[kQ2]);
  q = fma(s, q, kBm[kQ1]);
  q = fma(s, q, kBm[kQ0]);
  const double ed = (double)e;
  const double shi = fma(ed, kBm[kM2Ln2Hi], hi);               // exact: both on the 2^-42 grid
  const double slo = fma(ed, kBm[kM2Ln2Lo], lo);
  return shi + (s + fma(s2, q, slo));
}

// sin and cos of th in [0, 2 pi) by table: j = rint(256 th / pi), r = th - j pi/256 (pi/256 in three
// parts, the first two products exact), |r| <= pi/512, Taylor sin r / cos r to degree 5 / 4, and
// sin th = S_j cos r + C_j sin r, cos th = C_j cos r - S_j sin r with the correctly rounded
// S_j, C_j of kBmSinCosTab (513 rows; exact zeros at multiples of pi/2: no cancellation where sin
// or cos vanishes).  15 FP64 operations + one 16-byte load; <= 3.3e-16 relative
// (scripts/gen_bm_tables.py --check).
// Table: SCREP = 0 reads kBmSinCosTab through L1 (__ldg); SCREP > 0 reads a shared-memory copy
// replicated SCREP times, row j copy c at doubles [2 (j SCREP + c), +1], tab = this lane's copy
// (lane mod SCREP): a quarter-warp's 8 lanes then read 8 different copies -- 128 contiguous bytes,
// no bank conflict -- where the L1 gather of random rows cost ~8 wavefronts per request.
constexpr int kScRep = 8;
constexpr int kScTabRepBytes = (kBmSinCosN + 1) * kScRep * 16;   // 64.1 KB

__device__ __forceinline__ void bm_fill_sctab(double* smem_tab) {
  for (int i = threadIdx.x; i < (kBmSinCosN + 1) * kScRep * 2; i += blockDim.x)
    smem_tab[i] = (&kBmSinCosTab[0][0])[2 * (i / (2 * kScRep)) + (i & 1)];
}

template <int SCREP>
__device__ __forceinline__ void bm_sincos(double th, double& s, double& c, const double* __restrict__ sctab) {
  const double kr = fma(th, kBm[kSCInv], kBm[kRound]);      // 1.5 2^52 + rint(256 th / pi)
  const double kd = kr - kBm[kRound];
  double r = fma(-kd, kBm[kSCPi_0], th);
  r = fma(-kd, kBm[kSCPi_1], r);
  r = fma(-kd, kBm[kSCPi_2], r);
  const int j = __double2loint(kr) & 0x3FF;                  // 0..512
  double2 t;
  if constexpr (SCREP == 0) t = __ldg(reinterpret_cast<const double2*>(&kBmSinCosTab[j][0]));
  else t = *reinterpret_cast<const double2*>(sctab + 2 * SCREP * j);
  const double z = r * r;
  const double sr = fma(z * r, fma(z, kBm[kT5], kBm[kT3]), r);
  const double cr = fma(z, fma(z, kBm[kU4], kBm[kU2]), 1.0);
  s = fma(t.x, cr, t.y * sr);
  c = fma(t.y, cr, -(t.x * sr));
}

// sqrt(x) for x in [0, 75] to ~1 ulp: rsqrt approximation refined by one Goldschmidt step and one
// Newton correction (x = -0 or +0 returns x, like sqrt).
__device__ __forceinline__ double bm_sqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double s = x * y, h = 0.5 * y;
  const double e = fma(-s, h, 0.5);
  s = fma(s, e, s);
  h = fma(h, e, h);
  const double r = fma(-s, s, x);
  s = fma(r, h, s);
  return x == 0.0 ? x : s;
}

// The Box-Muller pair of block x; logtab / STRIDE as for bm_m2log_u53, sctab / SCREP as for bm_sincos.
template <int STRIDE, int SCREP = 0>
__device__ __forceinline__ void gaussian_pair_fast(const uint4 x, const double* __restrict__ logtab,
                                                   const double* __restrict__ sctab, double& g0, double& g1) {
  const unsigned long long k1 = (((unsigned long long)x.x << 32) | x.y) >> 11;
  const unsigned long long k2 = (((unsigned long long)x.z << 32) | x.w) >> 11;
  // u1 = (k1 + 1) 2^-53 and u2 = k2 2^-53 are never formed: -2 log u1 takes the integer with an
  // exponent bias, and th = u2 fl(2 pi) = k2 (2^-53 fl(2 pi)) is the same single rounding.
  const double rho = bm_sqrt(bm_m2log_u53<STRIDE>(__ull2double_rn(k1 + 1ull), logtab));
  const double th = __dmul_rn(__ull2double_rn(k2), kBm[kTwoPi53]);
  double s, c;
  bm_sincos<SCREP>(th, s, c, sctab);
  g0 = __dmul_rn(rho, c);
  g1 = __dmul_rn(rho, s);
}

}  // namespace sk
