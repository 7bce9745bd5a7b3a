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

// The same value without an int->double conversion (exponent-OR construction), kept for
// reference: with b = bit 52 of k and r = k mod 2^52, |S| = r'·2^-52 + 2^-53 where
// r' = b ? r : (2^52 - 1 - r); M = 1 + r'·2^-52 is built from bits and |S| = M - (1 - 2^-53)
// exactly (Sterbenz).  S = b ? |S| : -|S|.
__device__ __forceinline__ double uniform53_bits(uint32_t xa, uint32_t xb) {
  const uint32_t lo = __funnelshift_r(xb, xa, 11);          // bits 31..0 of k
  const uint32_t hi = xa >> 11;                             // bits 52..32 of k
  const uint32_t nb = ~(uint32_t)((int32_t)xa >> 31);       // all ones iff b == 0
  const uint32_t mlo = lo ^ nb;
  const uint32_t mhi = ((hi ^ nb) & 0x000FFFFFu) | 0x3FF00000u;
  const double M = __hiloint2double((int)mhi, (int)mlo);
  const double mag = __dsub_rn(M, __longlong_as_double(0x3FEFFFFFFFFFFFFFll));  // M - (1 - 2^-53)
  return __hiloint2double(__double2hiint(mag) ^ (int)(nb & 0x80000000u), __double2loint(mag));
}

// 2*pi rounded to the nearest double, 0x1.921fb54442d18p+2.
__device__ __forceinline__ double two_pi_f64() { return __longlong_as_double(0x401921FB54442D18ll); }

// Box-Muller pair from one block: u1 = (k1 + 1) 2^-53 in (0, 1], u2 = k2 2^-53 in [0, 1),
// rho = sqrt(-2 ln u1), th = u2 * fl(2 pi); (g0, g1) = (rho cos th, rho sin th).
// Full-precision libdevice log / sincos (no fast-math); single IEEE ops elsewhere.
__device__ __forceinline__ void gaussian_pair(const uint4 x, double& g0, double& g1) {
  const unsigned long long k1 = (((unsigned long long)x.x << 32) | x.y) >> 11;
  const unsigned long long k2 = (((unsigned long long)x.z << 32) | x.w) >> 11;
  const double u1 = __dmul_rn(__ull2double_rn(k1 + 1ull), 0x1p-53);
  const double u2 = __dmul_rn(__ull2double_rn(k2), 0x1p-53);
  const double rho = __dsqrt_rn(__dmul_rn(-2.0, log(u1)));
  const double th = __dmul_rn(u2, two_pi_f64());
  double s, c;
  sincos(th, &s, &c);
  g0 = __dmul_rn(rho, c);
  g1 = __dmul_rn(rho, s);
}

}  // namespace sk
