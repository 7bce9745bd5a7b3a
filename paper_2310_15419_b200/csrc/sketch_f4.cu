// sketch_f4.cu -- ±1 sketch of fp64 values on the 5th-gen tensor cores with packed fp4 operands
// (tcgen05.mma kind::mxf4, block-scaled e2m1, f32 accumulation in TMEM), sm_100a.
//
// Per column k, Â[:, k] = S[:, J_k] · a_k (Algorithm 3's inner loops) is computed
// EXACTLY on the tensor cores:
//  * signs -> fp4.  S[i, p] = ±1 is the e2m1 nibble 0x2 (+1.0) / 0xA (-1.0): the sign bit of the
//    nibble IS the Philox bit (bit 1 -> -1, include/sketch.h).  Operand A = S tile, M = 128 rows
//    x K = 64 nonzeros, K-major, packed 2 per byte (0.5 byte per (row, nonzero)).
//  * values -> binary signed digits.  With E = frexp exponent of max_p |a_p| of the column,
//    A_p = rint(a_p 2^(61-E)) (|A_p| <= 2^61, rounding is the only approximation: <= 2^-62 L max|a|)
//    and U_p = A_p + 2^63 (mod 2^64), the digits d_{p,s} = 2 bit_s(U_p) - 1 in {±1} satisfy
//    Σ_s d_{p,s} 2^s = 2 A_p + 1.  Operand B = 72 x 64 fp4: rows s < 64 hold d_{.,s}, row 64 is all
//    +1 (gives Σ_p S[i,p]), rows 65..71 are 0.
//  * D[i, s] = Σ_p S[i,p] d_{p,s} are integers with |D| <= L < 2^24: exact in f32.
//    Â[i] = 2^(E-62) (Σ_s 2^s D[i,s] - D[i,64]), formed with two exact int64 partial sums.
//  * both operands are produced by the same path: a Philox4x32-10 block (one nonzero x 128 rows)
//    or a value's 64-bit U, 32 x 32 bit-transposed across the warp (5 shuffle stages on lane-rotated
//    words), expanded to
//    nibbles ((y << (3-c)) & 0x88888888) | 0x22222222 and stored with STS.128 into the canonical
//    K-major no-swizzle layout (8-row x 16-byte core matrices).  Inside each 32-nonzero K chunk,
//    word c nibble n holds nonzero 4n + c for both A and B.
//  * CTA = up to 12 A-producer warps (tile = w % T, nonzero half = w / T) + 2 B-producer warps +
//    1 MMA warp; 2-stage smem ring, each stage kF4Sub = 3 K-steps (A: T x 12 KB, B: 3 x 2.5 KB) with mbarrier
//    full/empty (fewer, larger handshakes: 10.9 -> 8.4 ms on c5);
//    block scale factors (ue8m0 = 1.0) live in TMEM columns [448, 512).
// Measured (scripts/microbench_mxf4.cu): one M=128,K=64 mxf4 MMA reads its 4 KB A tile at
// ~44.5 B/clk -> ~89 entries/clk/SM, vs ~62 for int8 and 64 lanes/clk/SM for FP64 DFMA.
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "kernels.h"
#include "philox.cuh"

namespace sk {
namespace {

constexpr int kF4Tiles = 6;                       // 128-row tiles per CTA (max)
constexpr int kF4AWarps = 2 * kF4Tiles;          // A producers: (tile, nonzero half)
// B producers: nonzero half h, all 64 digit rows (4 warps with 32 rows each measured slower: c5
// 7.58 vs 7.24 ms)
constexpr int kF4BWarps = 2;
constexpr int kF4Producers = kF4AWarps + kF4BWarps;
constexpr int kF4LoaderWarp = kF4Producers;       // streams rowidx / vals into a smem ring
constexpr int kF4MmaWarp = kF4Producers + 1;
constexpr int kF4Threads = (kF4Producers + 2) * 32;
constexpr int kF4N = 72;                          // 64 digit rows + ones row + 7 zero rows
constexpr int kF4Ones = 64;
#ifndef SK_F4_SUB
#define SK_F4_SUB 3                               // (4 at ptxas -O3; at -O1 3 measured 7.31 vs 7.35 ms)
#define SK_F4_STAGES 2
#endif
constexpr int kF4Sub = SK_F4_SUB;                 // K-steps (64 nonzeros each) per smem stage
constexpr int kF4Stages = SK_F4_STAGES;
#ifndef SK_F4_JDEPTH
#define SK_F4_JDEPTH 6                             // (2 slots: 7.23 ms; 3: 7.30, 4: 7.31, 1: 7.35 on c5)
#endif
constexpr int kF4JSlots = SK_F4_JDEPTH / kF4Sub;  // nonzero-stream ring: one slot = one smem stage (kF4Sub K-steps)
constexpr int kF4ATile = 128 * 32;                // 128 rows x 64 fp4 = 4 KB
constexpr int kF4BSub = 2560;                     // B tile slot per K-step: 10 row groups x 256 B (72 rows, padded)
constexpr int kF4ATileS = kF4Sub * kF4ATile;      // one tile's A data per stage
constexpr int kF4Stage = kF4Tiles * kF4ATileS + kF4Sub * kF4BSub;
constexpr uint32_t kF4SfCol = 448;                // scale factors: TMEM columns [448, 512)
// try_wait suspend-time hint (ns): a waiting warp sleeps until the phase completes instead of
// spinning through SYNCS / BRA / YIELD loops that take issue slots from the producers.
#ifndef SK_SUSPEND_NS
#define SK_SUSPEND_NS 1000000
#endif
constexpr uint32_t kSuspendNs = SK_SUSPEND_NS;

struct F4Shared {
  uint64_t full[kF4Stages];
  uint64_t empty[kF4Stages];
  uint64_t jfull[kF4JSlots];
  uint64_t jempty[kF4JSlots];
  uint64_t done;
  uint32_t js[kF4JSlots][64 * kF4Sub];
  double vs[kF4JSlots][64 * kF4Sub];
  uint32_t tmem_base;
  unsigned long long maxabs_bits;
  int32_t E;
  int32_t nonfinite;
};

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void f4_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(s_u32(bar)), "r"(count));
}
__device__ __forceinline__ void f4_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(s_u32(bar)) : "memory");
}
__device__ __forceinline__ void f4_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}"
      :: "r"(s_u32(bar)), "r"(parity), "r"(kSuspendNs) : "memory");
}

// K-major, no-swizzle smem descriptor: core matrix = 8 rows x 16 B; LBO = stride between the two
// 16-byte K chunks (128 B), SBO = stride between 8-row groups (256 B); version 1 (sm_100).
__device__ __forceinline__ uint64_t f4_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)(128u >> 4) << 16;
  d |= (uint64_t)(256u >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// Block-scaled instruction descriptor: A = B = E2M1 (MXF4 format 1), K-major, D = F32,
// scale format E8M0, M = 128, N = 72, K = 64.
__host__ __device__ constexpr uint32_t f4_idesc() {
  return (1u << 7) | (1u << 10) | ((uint32_t)(kF4N >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);
}

// 32 x 32 bit transpose of NW independent word sets across the warp: on entry lane p holds word p
// (bit b = row b), on exit lane r holds row r (bit c = word c).  Between the two rotations every
// word is kept rotated left by its lane index, which makes each butterfly stage one SHFL + one
// LOP3 (the partner's word arrives already aligned): 2 + 5 ALU ops per word instead of 5 x 2.
// Stage s (distance j = 16 >> s) keeps rot(m_j, lane) in the lower lane of a pair, the
// complement in the upper lane.
template <int NW, int NS = 5>
__device__ __forceinline__ void f4_transpose(uint32_t (&x)[NW], int lane) {
  const uint32_t m[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int k = 0; k < NW; ++k) x[k] = __funnelshift_l(x[k], x[k], lane);
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const uint32_t rm = __funnelshift_l(m[s], m[s], lane);
    const uint32_t keep = (lane & (16 >> s)) ? ~rm : rm;
    uint32_t y[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) y[k] = __shfl_xor_sync(0xFFFFFFFFu, x[k], 16 >> s);
#pragma unroll
    for (int k = 0; k < NW; ++k)
      asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(x[k]) : "r"(x[k]), "r"(y[k]), "r"(keep));   // (x & keep) | (y & ~keep)
  }
#pragma unroll
  for (int k = 0; k < NW; ++k) x[k] = __funnelshift_r(x[k], x[k], lane);
}

// As f4_transpose, with the per-stage keep masks precomputed (loop-invariant per lane).
template <int NW, int NS>
__device__ __forceinline__ void f4_transpose_k(uint32_t (&x)[NW], int lane, const uint32_t (&keep)[4]) {
#pragma unroll
  for (int k = 0; k < NW; ++k) x[k] = __funnelshift_l(x[k], x[k], lane);
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    uint32_t y[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) y[k] = __shfl_xor_sync(0xFFFFFFFFu, x[k], 16 >> s);
#pragma unroll
    for (int k = 0; k < NW; ++k)
      asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(x[k]) : "r"(x[k]), "r"(y[k]), "r"(keep[s]));
  }
#pragma unroll
  for (int k = 0; k < NW; ++k) x[k] = __funnelshift_r(x[k], x[k], lane);
}

// 32 sign bits (bit l = nonzero l of the chunk; 1 -> -1.0) -> 16 bytes of e2m1 nibbles; word c
// nibble n holds nonzero 4n + c.
__device__ __forceinline__ uint32_t f4_valid_mask(int c, int nvalid) {
  // nibbles n with 4n + c < nvalid
  const int cnt = nvalid > c ? (nvalid - c + 3) >> 2 : 0;   // number of valid nibbles (0..8)
  return cnt >= 8 ? 0xFFFFFFFFu : ((1u << (4 * cnt)) - 1u);
}

__device__ __forceinline__ uint32_t f4_nib(uint32_t t) {   // (t & 0x88888888) | 0x22222222
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(t), "r"(0x88888888u), "r"(0x22222222u));
  return r;
}

[[maybe_unused]] __device__ __forceinline__ void f4_store_row(uint32_t addr, uint32_t y) {
  const uint32_t w0 = f4_nib(y << 3), w1 = f4_nib(y << 2), w2 = f4_nib(y << 1), w3 = f4_nib(y);
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" :: "r"(addr), "r"(w0), "r"(w1), "r"(w2), "r"(w3) : "memory");
}

// B rows: as f4_store_row, with nibbles of nonzeros >= nvalid (padding past the column end)
// forced to 0.0 so padded K positions contribute nothing whatever the S nibbles are.
__device__ __forceinline__ void f4_store_row_masked(uint32_t addr, uint32_t y, int nvalid) {
  uint32_t w0 = f4_nib(y << 3), w1 = f4_nib(y << 2), w2 = f4_nib(y << 1), w3 = f4_nib(y);
  if (nvalid < 32) {
    w0 &= f4_valid_mask(0, nvalid);
    w1 &= f4_valid_mask(1, nvalid);
    w2 &= f4_valid_mask(2, nvalid);
    w3 &= f4_valid_mask(3, nvalid);
  }
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" :: "r"(addr), "r"(w0), "r"(w1), "r"(w2), "r"(w3) : "memory");
}

// byte offset of row m, K chunk h inside a K-major no-swizzle tile (core matrices 8 x 16 B)
__device__ __forceinline__ uint32_t f4_off(int m, int h) {
  return (uint32_t)((m >> 3) * 256 + h * 128 + (m & 7) * 16);
}

// dbg (SKETCH_F4_DEBUG; tuning only, results invalid when nonzero), bit flags: 1 = no S stores,
// 2 = no MMAs, 4 = no proxy fences, 8 = no digit stores, 16 = no column scan, 32 = S warps skip
// Philox and the transposes, 64 = MMAs with N = 8.
// The debug switches exist only in builds with -DSK_F4_DEBUG=1 (the default build has none, so
// they cannot perturb the schedule of the production kernel).
#ifndef SK_F4_DEBUG
#define SK_F4_DEBUG 0
#endif
__global__ void __launch_bounds__(kF4Threads, 1) sk_rad_f4_kernel(const ApplyArgs P, const TcItem* items, int dbg_arg) {
  const int dbg = SK_F4_DEBUG ? dbg_arg : 0;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* stages = smem_raw + ((1024u - (s_u32(smem_raw) & 1023u)) & 1023u);
  F4Shared& sh = *reinterpret_cast<F4Shared*>(stages + kF4Stages * kF4Stage);
  const TcItem it = items[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t pb = P.colptr[it.col], pe = P.colptr[it.col + 1];
  if (it.pad) {   // last-wave item split along K: pad 1 = first half of the K-steps, 2 = second half
    const int64_t half = ((((pe - pb) + 63) >> 6) >> 1) << 6;
    if (it.pad == 1) pe = pb + half; else pb += half;
  }
  const int64_t L = pe - pb;
  const int nsteps = (int)((L + 63) >> 6);
  const int nsup = (nsteps + kF4Sub - 1) / kF4Sub;
  const int T = it.ntiles;                         // <= kF4Tiles
  const double* vals = reinterpret_cast<const double*>(P.vals);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kF4Stages; ++s) { f4_mbar_init(&sh.full[s], 2 * T + kF4BWarps); f4_mbar_init(&sh.empty[s], 1); }
    for (int s = 0; s < kF4JSlots; ++s) { f4_mbar_init(&sh.jfull[s], 32); f4_mbar_init(&sh.jempty[s], 2 * T + kF4BWarps); }
    f4_mbar_init(&sh.done, 1);
    sh.maxabs_bits = 0ull;
    sh.nonfinite = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kF4MmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(s_u32(&sh.tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // B rows kF4Ones.. of every stage are constant: the ones row = +1.0 (0x2), the 7 rows after it 0
  for (int i = threadIdx.x; i < kF4Stages * kF4Sub * 8 * 2; i += blockDim.x) {
    const int s = i / (16 * kF4Sub), sub = (i / 16) % kF4Sub, row = kF4Ones + (i % 16) / 2, h = i & 1;
    const uint32_t v = row == kF4Ones ? 0x22222222u : 0u;
    const uint32_t a = s_u32(stages + s * kF4Stage + kF4Tiles * kF4ATileS + sub * kF4BSub) + f4_off(row, h);
    asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" :: "r"(a), "r"(v) : "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const uint32_t tmem = sh.tmem_base;

  // scale factors = 1.0 (ue8m0 0x7F) in TMEM columns [448, 512), all 128 lanes
  if (warp < 4) {
    const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + kF4SfCol;
    const uint32_t v = 0x7F7F7F7Fu;
#pragma unroll
    for (int c = 0; c < 64; c += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};"
                   :: "r"(taddr + c), "r"(v) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  // column scale E (all producers)
  if (warp < kF4Producers && !(dbg & 16)) {
    unsigned long long mx = col_absmax_bits(vals, pb, pe, threadIdx.x, kF4Producers * 32);
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    if (lane == 0) atomicMax(&sh.maxabs_bits, mx);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double m = __longlong_as_double((long long)sh.maxabs_bits);
    int e = 0;
    if (isfinite(m)) frexp(m, &e); else sh.nonfinite = 1;
    sh.E = e;
  }
  __syncthreads();
  const int E = sh.E;

  if (warp < 2 * T) {
    // ===================== A producers: S tile (w % T), nonzero half, K-step class =====================
    // (kc = warp / 2T is 0 for every producer warp, but ptxas -O1 schedules the loop below measurably
    // better with it in the smem addresses: c5 7.23 vs 7.37 ms, same results; SASS-compared builds)
    const int t = warp % T, h = (warp / T) & 1, kc = warp / (2 * T);
    constexpr int kMine = kF4Sub;                    // K-steps of a stage this warp produces
    const uint32_t q = (uint32_t)(it.tile0 + t);
    // One smem stage holds kF4Sub K-steps: the warp generates all of them (independent Philox
    // chains, 4 kF4Sub interleaved 32x32 transposes) and signals the stage once.  Their row indices
    // come from one ring slot (one wait, one release per stage; padding past the column end was
    // zero-filled by the loader).
    const int jl = 32 * h + lane;
    for (int ss = 0; ss < nsup; ++ss) {
      const int stage = ss % kF4Stages, use = ss / kF4Stages;
      const int jslot = ss % kF4JSlots;
      f4_wait(&sh.jfull[jslot], (ss / kF4JSlots) & 1);
      uint32_t jv[kMine];
#pragma unroll
      for (int i = 0; i < kMine; ++i) jv[i] = sh.js[jslot][64 * (kc + i) + jl];
      __syncwarp();
      if (lane == 0) f4_arrive(&sh.jempty[jslot]);   // one arrival per warp
      uint32_t x[4 * kMine];
#pragma unroll
      for (int i = 0; i < kMine; ++i) {
        const uint32_t j = jv[i];
        const uint4 xb = (dbg & 32) ? make_uint4(j, j ^ 1u, j ^ 2u, j ^ 3u)
                                    : s_block(q, (uint64_t)P.row_offset + j, P.keys);   // padded nonzeros: B = 0
        x[4 * i + 0] = xb.x; x[4 * i + 1] = xb.y; x[4 * i + 2] = xb.z; x[4 * i + 3] = xb.w;
      }
      if (!(dbg & 32)) f4_transpose<4 * kMine>(x, lane);   // lane r: row 32qq + r over 32 nonzeros
      if (use > 0) f4_wait(&sh.empty[stage], (use - 1) & 1);
      if (!(dbg & 1)) {
        const uint32_t tile = s_u32(stages + stage * kF4Stage) + (uint32_t)(t * kF4ATileS) + f4_off(lane, h);
#pragma unroll
        for (int i = 0; i < kMine; ++i)
#pragma unroll
          for (int qq = 0; qq < 4; ++qq)   // row 32qq + lane
            f4_store_row(tile + (uint32_t)((kc + i) * kF4ATile + qq * 4 * 256), x[4 * i + qq]);
      }
      if (!(dbg & 4)) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) f4_arrive(&sh.full[stage]);
    }
  } else if (warp >= kF4AWarps && warp < kF4Producers) {
    // ===================== B producers: digits of nonzero half h =====================
    const int h = warp - kF4AWarps;
    // 2^(61-E) as two exact power-of-two factors (each within the double range)
    const int e1 = 61 - E > 1000 ? 1000 : (61 - E < -1000 ? -1000 : 61 - E);
    const double sc1 = ldexp(1.0, e1), sc2 = ldexp(1.0, 61 - E - e1);
    for (int ss = 0; ss < nsup; ++ss) {
      const int stage = ss % kF4Stages, use = ss / kF4Stages;
      uint32_t x[2 * kF4Sub];
      int nval[kF4Sub];
      const int jslot = ss % kF4JSlots;
      f4_wait(&sh.jfull[jslot], (ss / kF4JSlots) & 1);
      double vv[kF4Sub];
#pragma unroll
      for (int sub = 0; sub < kF4Sub; ++sub) vv[sub] = sh.vs[jslot][64 * sub + 32 * h + lane];
      __syncwarp();
      if (lane == 0) f4_arrive(&sh.jempty[jslot]);
#pragma unroll
      for (int sub = 0; sub < kF4Sub; ++sub) {
        const int ks = kF4Sub * ss + sub;
        const double v0 = vv[sub];
        const int64_t c0 = pb + (int64_t)ks * 64 + 32 * h;
        nval[sub] = (int)(pe - c0 < 0 ? 0 : (pe - c0 > 32 ? 32 : pe - c0));
        // U = A + 2^63 (mod 2^64); digit s = +1 iff bit s of U; nibble sign = NOT bit.  Padding
        // nonzeros past the column end contribute nothing: their B nibbles are 0.0 (masked below).
        unsigned long long U = 0ull;
        if (lane < nval[sub]) {
          const long long A = __double2ll_rn((v0 * sc1) * sc2);
          U = (unsigned long long)A ^ 0x8000000000000000ull;
        }
        x[2 * sub] = ~(uint32_t)U;                 // sign bits of the digit nibbles
        x[2 * sub + 1] = ~(uint32_t)(U >> 32);
      }
      f4_transpose<2 * kF4Sub>(x, lane);           // lane r: bit r (and 32 + r) of U per K-step
      if (use > 0) f4_wait(&sh.empty[stage], (use - 1) & 1);
      if (!(dbg & 8)) {
#pragma unroll
        for (int sub = 0; sub < kF4Sub; ++sub) {
          const uint32_t bt = s_u32(stages + stage * kF4Stage + kF4Tiles * kF4ATileS + sub * kF4BSub);
          f4_store_row_masked(bt + f4_off(lane, h), x[2 * sub], nval[sub]);
          f4_store_row_masked(bt + f4_off(32 + lane, h), x[2 * sub + 1], nval[sub]);
          if (nval[sub] < 32 && lane == 0) {   // partial (last) K chunk: the ones row too
            const uint32_t z = 0u;              // (y = 0 -> nibbles 0x2 = +1.0)
            f4_store_row_masked(bt + f4_off(kF4Ones, h), z, nval[sub]);
          }
        }
      }
      if (!(dbg & 4)) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) f4_arrive(&sh.full[stage]);
    }
  } else if (warp == kF4LoaderWarp) {
    // ===================== loader: rowidx / vals -> smem ring with cp.async ====================
    // Non-blocking: each lane issues its copies (zero-filled past the column end) and a
    // cp.async.mbarrier.arrive.noinc that fires when they land; it only blocks on ring space.
    for (int ss = 0; ss < nsup; ++ss) {
      const int slot = ss % kF4JSlots, use = ss / kF4JSlots;
      if (use > 0) f4_wait(&sh.jempty[slot], (use - 1) & 1);
#pragma unroll
      for (int e = 0; e < 2 * kF4Sub; ++e) {
        const int64_t p = pb + (int64_t)ss * (64 * kF4Sub) + 32 * e + lane;
        const bool ok = p < pe;
        const int64_t ps = ok ? p : pb;                 // any valid address; 0 bytes read (zero fill) if !ok
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;"
                     :: "r"(s_u32(&sh.js[slot][32 * e + lane])), "l"(P.rowidx + ps), "r"(ok ? 4 : 0) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;"
                     :: "r"(s_u32(&sh.vs[slot][32 * e + lane])), "l"(vals + ps), "r"(ok ? 8 : 0) : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" :: "r"(s_u32(&sh.jfull[slot])) : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (warp == kF4MmaWarp) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // (debug flag 64: N = 8, i.e. the MMAs read 256 B of the digits operand instead of 2304)
      const uint32_t idesc = (dbg & 64) ? ((f4_idesc() & ~(0x3Fu << 17)) | (1u << 17)) : f4_idesc();
      for (int ss = 0; ss < nsup; ++ss) {
        const int stage = ss % kF4Stages;
        f4_wait(&sh.full[stage], (ss / kF4Stages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t sb = s_u32(stages + stage * kF4Stage);
        for (int sub = 0; sub < kF4Sub; ++sub) {
          const int ks = kF4Sub * ss + sub;
          if (ks >= nsteps) break;
          const uint64_t bdesc = f4_desc(sb + kF4Tiles * kF4ATileS + sub * kF4BSub);
          for (int tt = 0; tt < T && !(dbg & 2); ++tt) {
            const uint64_t adesc = f4_desc(sb + tt * kF4ATileS + sub * kF4ATile);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}"
                :: "r"(tmem + (uint32_t)(tt * kF4N)), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(ks > 0 ? 1u : 0u),
                   "r"(tmem + kF4SfCol), "r"(tmem + kF4SfCol + 32u));
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     :: "r"(s_u32(&sh.empty[stage])) : "memory");
      }
      if (nsteps > 0)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     :: "r"(s_u32(&sh.done)) : "memory");
    }
    __syncwarp();
  }

  // ===================== epilogue: warps 0..11 read D (lane quarter = warp % 4) =====================
  if (warp < kF4Producers) {
    if (nsteps > 0) {
      f4_wait(&sh.done, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    const int qw = warp & 3;
    double* outc = reinterpret_cast<double*>(P.out) + (int64_t)it.col * P.ld;
    const double nan = __longlong_as_double(0x7FF8000000000000ll);
    for (int tt = warp >> 2; warp < 12 && tt < T; tt += 3) {
      long long lo = 0, hi = 0, ones = 0;
      if (nsteps > 0) {
        const uint32_t base = tmem + ((uint32_t)(32 * qw) << 16) + (uint32_t)(tt * kF4N);
#pragma unroll
        for (int c = 0; c < kF4N; c += 8) {
          uint32_t D[8];
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                       : "=r"(D[0]), "=r"(D[1]), "=r"(D[2]), "=r"(D[3]), "=r"(D[4]), "=r"(D[5]), "=r"(D[6]), "=r"(D[7])
                       : "r"(base + (uint32_t)c));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const long long dv = (long long)__float2ll_rn(__uint_as_float(D[u]));
            const int s = c + u;
            if (s < 32) lo += dv << s;
            else if (s < 64) hi += dv << (s - 32);
            else if (s == 64) ones = dv;
          }
        }
      }
      const int64_t row = (int64_t)(it.tile0 + tt) * 128 + 32 * qw + lane;
      if (row < P.d) {
        // Σ_s 2^s D_s - D_64 = hi 2^32 + (lo - ones), both parts exact in fp64; one rounding
        const double v = scalbn((double)hi * 4294967296.0 + (double)(lo - ones), E - 62);
        // a column holding a NaN / Inf (the digits need finite values) is marked NaN here and
        // rewritten with the IEEE result by sk_f4_ieee_fixup_kernel
        const double res = sh.nonfinite ? nan : v;
        // K-split halves add into the zeroed output: 0 + a + b rounds the same in either order
        if (it.pad) atomicAdd(outc + row, res); else outc[row] = res;
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  __syncthreads();
  if (warp == kF4MmaWarp) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(512));
  }
}

// ============================================================================================
// Persistent variant (the default when the items fill more than one wave; sketch_set_f4_persistent /
// SKETCH_F4_PERSIST): one CTA per SM; its first item is blockIdx.x, the next ones come from a global
// counter claimed by the scan warp (dynamic, like the hardware scheduler).  TMEM, the barriers, the
// constant B rows and the scale factors are set up once; the scan warp computes the next item's
// column scale E while the current item runs (2-slot ring; the whole CTA scans item 0); the A
// producers produce the first stage of item k before they read out item k-1's accumulators, so the
// MMA warp restarts as soon as TMEM is free (tfree) with a stage already waiting.  All roles walk
// the same global stage sequence g (ring slot g % 2, phase g / 2); A warps without a tile in an
// item (T < 6) skip it and wait for its accumulators, and the B warps arrive on the stage barriers
// in their place.
// 4 K-steps per smem stage (2 stages of 6 x 16 KB + 4 x 2.5 KB): more independent Philox chains per
// producer warp between two handshakes (c5 7.155 -> 7.085 ms; the per-item kernel keeps 3, which it
// measured faster at ptxas -O1: 7.31 vs 7.35 ms)
constexpr int kF4PSub = 4;
#ifndef SK_F4P_OFFSPEC
#define SK_F4P_OFFSPEC 1                            // separate S-producer loop for row_offset == 0 (c5 7.00 -> 6.98 ms)
#endif
#ifndef SK_F4P_T4
#define SK_F4P_T4 1                                 // c5 7.10 -> 7.00 ms (scripts/gpurun/gpu_r2bo.sh)
#endif
// SK_F4P_T4: the S transpose stops one butterfly stage early.  Lane r then holds row r's bits at the
// positions of r's parity and row r^1's at the others (bit c <-> nonzero c, or c^1 for the other row),
// so each lane stores two 8-byte halves: the even-nonzero half of row pair k = lane/2 comes from the
// even lane, the odd half from the odd lane.  The 16-byte K chunk of a row holds its nibble words in
// the order c0, c2, c1, c3 (word c nibble n = nonzero 4n + c), for the digits operand too, and the
// logical rows 2k, 2k+1 sit in physical rows k, 16 + k of their 32-row group, so each 8-byte store of
// the warp fills 16 whole rows of two core matrices (no bank conflicts); the read-out maps TMEM lane
// l back to row 2l (l < 16) or 2(l - 16) + 1.
// digits rows in the chunk word order c0, c2, c1, c3 (SK_F4P_T4)
__device__ __forceinline__ void f4p_store_row_masked_perm(uint32_t addr, uint32_t y, int nvalid) {
  uint32_t w0 = f4_nib(y << 3), w1 = f4_nib(y << 2), w2 = f4_nib(y << 1), w3 = f4_nib(y);
  if (nvalid < 32) {
    w0 &= f4_valid_mask(0, nvalid);
    w1 &= f4_valid_mask(1, nvalid);
    w2 &= f4_valid_mask(2, nvalid);
    w3 &= f4_valid_mask(3, nvalid);
  }
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" :: "r"(addr), "r"(w0), "r"(w2), "r"(w1), "r"(w3) : "memory");
}
__device__ __forceinline__ int f4p_row_of_lane(int l) { return SK_F4P_T4 ? (l < 16 ? 2 * l : 2 * (l - 16) + 1) : l; }
// The scan warp starts the next item's column scan when the running item has SK_F4P_SCANLEAD stages
// to go: started an item ahead, the scanned values (148 columns in flight) were evicted from L2
// before the loader read them, DRAM 699 MB per c5 launch; at 64 stages 627 MB (616 algorithmic) at
// the same time (scripts/gpurun/gpu_r2bj.sh).  0: scan as soon as the slot is free.
#ifndef SK_F4P_SCANLEAD
#define SK_F4P_SCANLEAD 64
#endif
constexpr int kF4PATileS = kF4PSub * kF4ATile;
constexpr int kF4PStage = kF4Tiles * kF4PATileS + kF4PSub * kF4BSub;
constexpr int kF4PJSlots = 2;                       // nonzero-stream ring: one slot = one smem stage
constexpr int kF4PScanWarp = kF4MmaWarp + 1;
constexpr int kF4PThreads = (kF4PScanWarp + 1) * 32;
constexpr int kF4PEpiWarps = kF4AWarps;            // epilogue: the 12 A warps (lane quarter = warp % 4)

struct F4PShared {
  uint64_t full[kF4Stages];
  uint64_t empty[kF4Stages];
  uint64_t jfull[kF4PJSlots];
  uint64_t jempty[kF4PJSlots];
  uint64_t done;                // MMA -> epilogue: one phase per item
  uint64_t tfree;               // epilogue -> MMA: accumulators read out, one phase per item
  uint64_t efull[2];            // scan warp -> B producers / epilogue: E of item k in slot k % 2
  uint64_t eempty[2];
  uint32_t js[kF4PJSlots][64 * kF4PSub];
  double vs[kF4PJSlots][64 * kF4PSub];
  int64_t item[2];              // item index of the CTA's item k in slot k % 2 (-1: no more items)
  unsigned long long mx0;       // max |a| bits of item 0 (scanned by the whole CTA)
  uint32_t loaded;              // stages the loader has issued (the scan warp starts item k + 1's scan late)
  int32_t E[2];
  int32_t nonfinite[2];
  uint32_t tmem_base;
};

struct F4PItem {
  int64_t pb, pe;
  int col, tile0, T, pad, nsteps, nsup;
};

__device__ __forceinline__ F4PItem f4p_item(const ApplyArgs& P, const TcItem* items, int64_t idx) {
  const TcItem it = items[idx];
  F4PItem r;
  r.pb = P.colptr[it.col];
  r.pe = P.colptr[it.col + 1];
  if (it.pad) {
    const int64_t half = ((((r.pe - r.pb) + 63) >> 6) >> 1) << 6;
    if (it.pad == 1) r.pe = r.pb + half; else r.pb += half;
  }
  r.col = it.col;
  r.tile0 = it.tile0;
  r.T = it.ntiles;
  r.pad = it.pad;
  r.nsteps = (int)((r.pe - r.pb + 63) >> 6);
  r.nsup = (r.nsteps + kF4PSub - 1) / kF4PSub;
  return r;
}

// max |v[p]| bits over [pb, pe) by one warp, 8 independent 16-byte loads in flight per lane
__device__ __forceinline__ unsigned long long f4p_scan(const double* __restrict__ v, int64_t pb, int64_t pe, int lane) {
  constexpr unsigned long long kAbs = 0x7FFFFFFFFFFFFFFFull;
  auto ab = [](double x) { return (unsigned long long)__double_as_longlong(x) & kAbs; };
  unsigned long long m[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  // first index >= pb whose address is 16-byte aligned (v is 8-byte aligned)
  int64_t a = pb + ((reinterpret_cast<uintptr_t>(v + pb) & 15) ? 1 : 0);
  if (a > pe) a = pe;
  const int64_t n2 = (pe - a) >> 1;
  if (lane == 0 && pb < a) m[0] = ab(__ldg(v + pb));
  if (lane == 31 && a + 2 * n2 < pe) m[1] = ab(__ldg(v + a + 2 * n2));
  const double2* v2 = reinterpret_cast<const double2*>(v + a);
  int64_t i = lane;
  for (; i + 7 * 32 < n2; i += 8 * 32) {
    double2 x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = __ldg(v2 + i + 32 * u);
#pragma unroll
    for (int u = 0; u < 8; ++u) m[u] = max(m[u], max(ab(x[u].x), ab(x[u].y)));
  }
  for (; i < n2; i += 32) {
    const double2 x = __ldg(v2 + i);
    m[0] = max(m[0], max(ab(x.x), ab(x.y)));
  }
  unsigned long long r = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) r = max(r, m[u]);
  for (int o = 16; o; o >>= 1) r = max(r, __shfl_xor_sync(0xFFFFFFFFu, r, o));
  return r;
}

static_assert(kF4Stages == 2 && kF4PJSlots == 2, "the persistent kernel indexes its rings with g & 1");
static_assert(kF4Stages * kF4PStage + 8192 <= 227 * 1024, "persistent kernel shared memory");

// A wait expected to last long (an item, or the rest of one): poll with explicit sleeps instead of
// the try_wait loop, whose ~40 ns suspensions cost the producers ~7% of an SMSP per waiting warp.
__device__ __forceinline__ void f4_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns) {
  for (;;) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(s_u32(bar)), "r"(parity) : "memory");
    if (ok) break;
    __nanosleep(ns);
  }
}

__device__ __forceinline__ void f4_arrive_cnt(uint64_t* bar, uint32_t cnt) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" :: "r"(s_u32(bar)), "r"(cnt) : "memory");
}

// One smem stage of S tile t (nonzero half h) for global stage g (as sk_rad_f4_kernel's A loop).
// kOff: the plan has a row offset (a row shard); without one the Philox counter's high word is 0
#ifndef SK_F4P_KEEP
#define SK_F4P_KEEP 1                               // transpose masks computed once per item (c5 6.977 -> 6.965 ms)
#endif
template <bool kOff>
__device__ __forceinline__ void f4p_a_stage(F4PShared& sh, unsigned char* stages, const PhiloxKeys& keys,
                                            uint64_t row_offset, uint32_t g, uint32_t q, int t, int h, int lane,
                                            const uint32_t (&keep)[4]) {
  constexpr int kMine = kF4PSub;
  const uint32_t stage = g & 1u, use = g >> 1, jslot = g & 1u;
  const int jl = 32 * h + lane;
  f4_wait(&sh.jfull[jslot], use & 1u);
  uint32_t jv[kMine];
#pragma unroll
  for (int i = 0; i < kMine; ++i) jv[i] = sh.js[jslot][64 * i + jl];
  __syncwarp();
  if (lane == 0) f4_arrive(&sh.jempty[jslot]);
  uint32_t x[4 * kMine];
#pragma unroll
  for (int i = 0; i < kMine; ++i) {
    const uint4 xb = s_block(q, kOff ? row_offset + jv[i] : (uint64_t)jv[i], keys);
    x[4 * i + 0] = xb.x; x[4 * i + 1] = xb.y; x[4 * i + 2] = xb.z; x[4 * i + 3] = xb.w;
  }
#if SK_F4P_T4
#if SK_F4P_KEEP
  f4_transpose_k<4 * kMine, 4>(x, lane, keep);
#else
  (void)keep;
  f4_transpose<4 * kMine, 4>(x, lane);
#endif
  if (use > 0) f4_wait(&sh.empty[stage], (use - 1) & 1u);
  const uint32_t base = s_u32(stages + stage * kF4PStage) + (uint32_t)(t * kF4PATileS) + 8u * (uint32_t)(lane & 1);
  const uint32_t ra = base + f4_off(lane >> 1, h), rb = base + f4_off(16 + (lane >> 1), h);
#pragma unroll
  for (int i = 0; i < kMine; ++i)
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      const uint32_t y = x[4 * i + qq], o = (uint32_t)(i * kF4ATile + qq * 4 * 256);
      asm volatile("st.shared.v2.b32 [%0], {%1, %2};" :: "r"(ra + o), "r"(f4_nib(y << 3)), "r"(f4_nib(y << 1)) : "memory");
      asm volatile("st.shared.v2.b32 [%0], {%1, %2};" :: "r"(rb + o), "r"(f4_nib(y << 2)), "r"(f4_nib(y)) : "memory");
    }
#else
  f4_transpose<4 * kMine>(x, lane);
  if (use > 0) f4_wait(&sh.empty[stage], (use - 1) & 1u);
  const uint32_t tile = s_u32(stages + stage * kF4PStage) + (uint32_t)(t * kF4PATileS) + f4_off(lane, h);
#pragma unroll
  for (int i = 0; i < kMine; ++i)
#pragma unroll
    for (int qq = 0; qq < 4; ++qq)
      f4_store_row(tile + (uint32_t)(i * kF4ATile + qq * 4 * 256), x[4 * i + qq]);
#endif
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) f4_arrive(&sh.full[stage]);
}

// Epilogue of item k (warps 0..11): wait for its accumulators, read TMEM, form Â, free TMEM.
// The ones row of B stays all +1.0 in the persistent kernel, so D[i, 64] also sums S over the padded
// K positions of the item's last K-step (nsteps 64 - L of them); the loader zero-filled their row
// index, so each is S[i, row_offset + 0], and D[i, 64] - pad S[i, row_offset] is the plain Σ_p S[i, p].
__device__ __forceinline__ void f4p_epilogue(F4PShared& sh, const ApplyArgs& P, const F4PItem& it, int64_t k,
                                             uint32_t tmem, int warp, int lane) {
  f4_wait_sleep(&sh.done, (uint32_t)(k & 1), 200);
  f4_wait(&sh.efull[k & 1], (uint32_t)((k >> 1) & 1));
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int E = sh.E[k & 1];
  const int nonfinite = sh.nonfinite[k & 1];
  const int qw = warp & 3;
  double* outc = reinterpret_cast<double*>(P.out) + (int64_t)it.col * P.ld;
  const double nan = __longlong_as_double(0x7FF8000000000000ll);
  for (int tt = warp >> 2; tt < it.T; tt += 3) {
    long long lo = 0, hi = 0, ones = 0;
    if (it.nsteps > 0) {
      const uint32_t base = tmem + ((uint32_t)(32 * qw) << 16) + (uint32_t)(tt * kF4N);
#pragma unroll
      for (int c = 0; c < kF4N; c += 8) {
        uint32_t D[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(D[0]), "=r"(D[1]), "=r"(D[2]), "=r"(D[3]), "=r"(D[4]), "=r"(D[5]), "=r"(D[6]), "=r"(D[7])
                     : "r"(base + (uint32_t)c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const long long dv = (long long)__float2ll_rn(__uint_as_float(D[u]));
          const int s = c + u;
          if (s < 32) lo += dv << s;
          else if (s < 64) hi += dv << (s - 32);
          else if (s == 64) ones = dv;
        }
      }
    }
    const int lrow = f4p_row_of_lane(lane);
    const int64_t row = (int64_t)(it.tile0 + tt) * 128 + 32 * qw + lrow;
    const int pad = it.nsteps * 64 - (int)(it.pe - it.pb);
    if (pad > 0) {
      const uint4 x0 = s_block((uint32_t)(it.tile0 + tt), (uint64_t)P.row_offset, P.keys);
      const uint32_t w = qw == 0 ? x0.x : qw == 1 ? x0.y : qw == 2 ? x0.z : x0.w;
      ones -= ((w >> lrow) & 1u) ? -(long long)pad : (long long)pad;   // bit 1 -> S = -1
    }
    if (row < P.d) {
      const double v = scalbn((double)hi * 4294967296.0 + (double)(lo - ones), E - 62);
      const double res = nonfinite ? nan : v;
      if (it.pad) atomicAdd(outc + row, res); else outc[row] = res;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    f4_arrive(&sh.tfree);
    f4_arrive(&sh.eempty[k & 1]);
  }
}

// Item k of this CTA, published by the scan warp (slot k % 2, with efull): -1 when there is none.
__device__ __forceinline__ int64_t f4p_next(F4PShared& sh, int64_t k) {
  f4_wait(&sh.efull[k & 1], (uint32_t)((k >> 1) & 1));
  return sh.item[k & 1];
}

__global__ void __launch_bounds__(kF4PThreads, 1) sk_rad_f4p_kernel(const ApplyArgs P, const TcItem* items, int64_t n_items,
                                                                     unsigned long long* next_item) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* stages = smem_raw + ((1024u - (s_u32(smem_raw) & 1023u)) & 1023u);
  F4PShared& sh = *reinterpret_cast<F4PShared*>(stages + kF4Stages * kF4PStage);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t G = gridDim.x;
  const double* vals = reinterpret_cast<const double*>(P.vals);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kF4Stages; ++s) { f4_mbar_init(&sh.full[s], kF4AWarps + kF4BWarps); f4_mbar_init(&sh.empty[s], 1); }
    for (int s = 0; s < kF4PJSlots; ++s) { f4_mbar_init(&sh.jfull[s], 32); f4_mbar_init(&sh.jempty[s], kF4AWarps + kF4BWarps); }
    f4_mbar_init(&sh.done, 1);
    f4_mbar_init(&sh.tfree, kF4PEpiWarps);
    for (int s = 0; s < 2; ++s) { f4_mbar_init(&sh.efull[s], 1); f4_mbar_init(&sh.eempty[s], kF4PEpiWarps + kF4BWarps); }
    sh.mx0 = 0ull;
    sh.loaded = 0u;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kF4MmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(s_u32(&sh.tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < kF4Stages * kF4PSub * 8 * 2; i += blockDim.x) {
    const int s = i / (16 * kF4PSub), sub = (i / 16) % kF4PSub, row = kF4Ones + (i % 16) / 2, h = i & 1;
    const uint32_t v = row == kF4Ones ? 0x22222222u : 0u;
    const uint32_t a = s_u32(stages + s * kF4PStage + kF4Tiles * kF4PATileS + sub * kF4BSub) + f4_off(row, h);
    asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" :: "r"(a), "r"(v) : "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const uint32_t tmem = sh.tmem_base;
  if (warp < 4) {
    const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + kF4SfCol;
    const uint32_t v = 0x7F7F7F7Fu;
#pragma unroll
    for (int c = 0; c < 64; c += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};"
                   :: "r"(taddr + c), "r"(v) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  {   // item 0's column scale: the whole CTA scans (later items: the scan warp, one item ahead)
    const F4PItem it0 = f4p_item(P, items, blockIdx.x);
    unsigned long long mx = col_absmax_bits(vals, it0.pb, it0.pe, threadIdx.x, kF4PThreads);
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    if (lane == 0) atomicMax(&sh.mx0, mx);
  }
  __syncthreads();

  if (warp < kF4AWarps) {
    // ===================== A producers + epilogue =====================
    // A warps without a tile in an item (T < 6) skip its stages (the B warps arrive for them) and
    // wait for the item's accumulators instead: a parity wait is only meaningful within one phase of
    // the barrier, so no warp may run more than one stage ahead of the ring.
    uint32_t g = 0;
    F4PItem prev{};
    bool pending = false;                          // prev's epilogue not done yet
    PhiloxKeys keys;                               // in per-thread registers across the item loop (a
#pragma unroll                                     // shuffle hides their uniformity, so they are not
    for (int r = 0; r < 10; ++r) {                 // re-read from the constant bank every stage)
      keys.k0[r] = __shfl_sync(0xFFFFFFFFu, P.keys.k0[r], lane);
      keys.k1[r] = __shfl_sync(0xFFFFFFFFu, P.keys.k1[r], lane);
    }
    const uint64_t row_offset = (uint64_t)P.row_offset;
    uint32_t keep[4];                              // the transpose's per-stage masks (this lane's)
#pragma unroll
    for (int st = 0; st < 4; ++st) {
      const uint32_t mm = st == 0 ? 0x0000FFFFu : st == 1 ? 0x00FF00FFu : st == 2 ? 0x0F0F0F0Fu : 0x33333333u;
      const uint32_t rm = __funnelshift_l(mm, mm, lane);
      keep[st] = (lane & (16 >> st)) ? ~rm : rm;
    }
    for (int64_t k = 0;; ++k) {
      const int64_t idx = f4p_next(sh, k);
      if (idx < 0) {
        if (pending) f4p_epilogue(sh, P, prev, k - 1, tmem, warp, lane);
        break;
      }
      const F4PItem it = f4p_item(P, items, idx);
      const int T = it.T;
      if (warp < 2 * T) {
        const int t = warp % T, h = (warp / T) & 1;
        const uint32_t q = (uint32_t)(it.tile0 + t);
        int ss = 0;
        if (it.nsup > 0) {   // the first stage of item k before item k-1's epilogue
          if (SK_F4P_OFFSPEC && row_offset == 0) f4p_a_stage<false>(sh, stages, keys, row_offset, g, q, t, h, lane, keep);
          else f4p_a_stage<true>(sh, stages, keys, row_offset, g, q, t, h, lane, keep);
          ++ss;
        }
        if (pending) f4p_epilogue(sh, P, prev, k - 1, tmem, warp, lane);
        if (SK_F4P_OFFSPEC && row_offset == 0)
          for (; ss < it.nsup; ++ss) f4p_a_stage<false>(sh, stages, keys, row_offset, g + (uint32_t)ss, q, t, h, lane, keep);
        else
          for (; ss < it.nsup; ++ss) f4p_a_stage<true>(sh, stages, keys, row_offset, g + (uint32_t)ss, q, t, h, lane, keep);
        pending = true;
      } else {
        if (pending) f4p_epilogue(sh, P, prev, k - 1, tmem, warp, lane);
        f4p_epilogue(sh, P, it, k, tmem, warp, lane);   // waits for item k's accumulators
        pending = false;
      }
      g += (uint32_t)it.nsup;
      prev = it;
    }
  } else if (warp < kF4Producers) {
    // ===================== B producers: digits of nonzero half h =====================
    const int h = warp - kF4AWarps;
    uint32_t g = 0;
    for (int64_t k = 0;; ++k) {
      const int64_t idx = f4p_next(sh, k);
      if (idx < 0) break;
      const F4PItem it = f4p_item(P, items, idx);
      const uint32_t cnt = 1u + (uint32_t)(kF4Tiles - it.T);   // own arrival + those of the idle A warps (12 - 2T)
      const int E = sh.E[k & 1];
      __syncwarp();
      if (lane == 0) f4_arrive(&sh.eempty[k & 1]);
      const int e1 = 61 - E > 1000 ? 1000 : (61 - E < -1000 ? -1000 : 61 - E);
      const double sc1 = ldexp(1.0, e1), sc2 = ldexp(1.0, 61 - E - e1);
      for (int ss = 0; ss < it.nsup; ++ss, ++g) {
        const uint32_t stage = g & 1u, use = g >> 1, jslot = g & 1u;
        uint32_t x[2 * kF4PSub];
        int nval[kF4PSub];
        f4_wait(&sh.jfull[jslot], use & 1u);
        double vv[kF4PSub];
#pragma unroll
        for (int sub = 0; sub < kF4PSub; ++sub) vv[sub] = sh.vs[jslot][64 * sub + 32 * h + lane];
        __syncwarp();
        if (lane == 0) f4_arrive_cnt(&sh.jempty[jslot], cnt);
#pragma unroll
        for (int sub = 0; sub < kF4PSub; ++sub) {
          const int ks = kF4PSub * ss + sub;
          const int64_t c0 = it.pb + (int64_t)ks * 64 + 32 * h;
          nval[sub] = (int)(it.pe - c0 < 0 ? 0 : (it.pe - c0 > 32 ? 32 : it.pe - c0));
          unsigned long long U = 0ull;
          if (lane < nval[sub]) {
            const long long A = __double2ll_rn((vv[sub] * sc1) * sc2);
            U = (unsigned long long)A ^ 0x8000000000000000ull;
          }
          x[2 * sub] = ~(uint32_t)U;
          x[2 * sub + 1] = ~(uint32_t)(U >> 32);
        }
        f4_transpose<2 * kF4PSub>(x, lane);
        if (use > 0) f4_wait(&sh.empty[stage], (use - 1) & 1u);
#pragma unroll
        for (int sub = 0; sub < kF4PSub; ++sub) {
          const uint32_t bt = s_u32(stages + stage * kF4PStage + kF4Tiles * kF4PATileS + sub * kF4BSub);
#if SK_F4P_T4
          f4p_store_row_masked_perm(bt + f4_off(lane, h), x[2 * sub], nval[sub]);
          f4p_store_row_masked_perm(bt + f4_off(32 + lane, h), x[2 * sub + 1], nval[sub]);
#else
          f4_store_row_masked(bt + f4_off(lane, h), x[2 * sub], nval[sub]);
          f4_store_row_masked(bt + f4_off(32 + lane, h), x[2 * sub + 1], nval[sub]);
#endif
          // (the ones row stays all +1.0: the padding's share of D[i, 64] is removed in the read-out)
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) f4_arrive_cnt(&sh.full[stage], cnt);
      }
    }
  } else if (warp == kF4LoaderWarp) {
    // ===================== loader: rowidx / vals -> smem ring =====================
    uint32_t g = 0;
    for (int64_t k = 0;; ++k) {
      const int64_t idx = f4p_next(sh, k);
      if (idx < 0) break;
      const F4PItem it = f4p_item(P, items, idx);
      for (int ss = 0; ss < it.nsup; ++ss, ++g) {
        const uint32_t slot = g & 1u, use = g >> 1;
        if (use > 0) f4_wait(&sh.jempty[slot], (use - 1) & 1u);
#pragma unroll
        for (int e = 0; e < 2 * kF4PSub; ++e) {
          const int64_t p = it.pb + (int64_t)ss * (64 * kF4PSub) + 32 * e + lane;
          const bool ok = p < it.pe;
          const int64_t ps = ok ? p : it.pb;
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;"
                       :: "r"(s_u32(&sh.js[slot][32 * e + lane])), "l"(P.rowidx + ps), "r"(ok ? 4 : 0) : "memory");
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;"
                       :: "r"(s_u32(&sh.vs[slot][32 * e + lane])), "l"(vals + ps), "r"(ok ? 8 : 0) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" :: "r"(s_u32(&sh.jfull[slot])) : "memory");
#if SK_F4P_SCANLEAD
        if (lane == 0) *reinterpret_cast<volatile uint32_t*>(&sh.loaded) = g + 1;
#endif
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (warp == kF4MmaWarp) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t idesc = f4_idesc();
      uint32_t g = 0;
      for (int64_t k = 0;; ++k) {
        const int64_t idx = f4p_next(sh, k);
        if (idx < 0) break;
        const F4PItem it = f4p_item(P, items, idx);
        if (k > 0) {   // item k-1's accumulators read out
          f4_wait(&sh.tfree, (uint32_t)((k - 1) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        for (int ss = 0; ss < it.nsup; ++ss, ++g) {
          const uint32_t stage = g & 1u;
          f4_wait(&sh.full[stage], (g >> 1) & 1u);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sb = s_u32(stages + stage * kF4PStage);
          for (int sub = 0; sub < kF4PSub; ++sub) {
            const int ks = kF4PSub * ss + sub;
            if (ks >= it.nsteps) break;
            const uint64_t bdesc = f4_desc(sb + kF4Tiles * kF4PATileS + sub * kF4BSub);
            for (int tt = 0; tt < it.T; ++tt) {
              const uint64_t adesc = f4_desc(sb + tt * kF4PATileS + sub * kF4ATile);
              asm volatile(
                  "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}"
                  :: "r"(tmem + (uint32_t)(tt * kF4N)), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(ks > 0 ? 1u : 0u),
                     "r"(tmem + kF4SfCol), "r"(tmem + kF4SfCol + 32u));
            }
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                       :: "r"(s_u32(&sh.empty[stage])) : "memory");
        }
        if (it.nsteps > 0)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                       :: "r"(s_u32(&sh.done)) : "memory");
        else
          f4_arrive(&sh.done);
      }
    }
    __syncwarp();
  } else {
    // ===================== scan warp: the CTA's next item and its column scale E, one item ahead ====
    // Item 0 is blockIdx.x; later items come from a global counter (dynamic: CTAs that drew shorter
    // items take more of them, as the hardware scheduler does for one CTA per item).
    uint32_t g_start = 0, nsup_prev = 0;           // stage range of item k - 1 (the one running)
    for (int64_t k = 0;; ++k) {
      if (k >= 2) f4_wait_sleep(&sh.eempty[k & 1], (uint32_t)(((k >> 1) - 1) & 1), 2000);
#if SK_F4P_SCANLEAD
      // scan item k while item k - 1 has its last SK_F4P_SCANLEAD stages to go (earlier, the scanned
      // values are evicted from L2 before the loader reads them)
      if (k >= 1 && nsup_prev > SK_F4P_SCANLEAD) {
        const uint32_t until = g_start + nsup_prev - SK_F4P_SCANLEAD;
        while (*reinterpret_cast<volatile uint32_t*>(&sh.loaded) < until) __nanosleep(500);
      }
#endif
      int64_t idx = blockIdx.x;
      if (k > 0) {
        unsigned long long v = 0;
        if (lane == 0) v = atomicAdd(next_item, 1ull);
        idx = G + (int64_t)__shfl_sync(0xFFFFFFFFu, v, 0);
      }
      if (idx >= n_items) idx = -1;
      unsigned long long mx = k == 0 ? sh.mx0 : 0ull;
      if (idx >= 0) {
        const F4PItem it = f4p_item(P, items, idx);
        if (k > 0) mx = f4p_scan(vals, it.pb, it.pe, lane);
        if (k > 0) g_start += nsup_prev;
        nsup_prev = (uint32_t)it.nsup;
      }
      if (lane == 0) {
        const double m = __longlong_as_double((long long)mx);
        int e = 0;
        int nf = 0;
        if (isfinite(m)) frexp(m, &e); else nf = 1;
        sh.item[k & 1] = idx;
        sh.E[k & 1] = e;
        sh.nonfinite[k & 1] = nf;
        f4_arrive(&sh.efull[k & 1]);
      }
      __syncwarp();
      if (idx < 0) break;
    }
  }
  __syncthreads();
  if (warp == kF4MmaWarp) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(512));
  }
}

}  // namespace

int f4_tiles_per_cta() {   // SKETCH_F4_TILES (tuning only): fewer row tiles per CTA
  static const int t = [] { const char* v = getenv("SKETCH_F4_TILES"); const int x = v ? atoi(v) : kF4Tiles;
                            return x >= 1 && x <= kF4Tiles ? x : kF4Tiles; }();
  return t;
}

// Zero the Â rows of the K-split items (pad == 1 marks the first half of each pair).
__global__ void sk_f4_zero_split_kernel(const ApplyArgs P, const TcItem* items) {
  const TcItem it = items[blockIdx.x];
  if (it.pad != 1) return;
  const int64_t r0 = (int64_t)it.tile0 * 128;
  const int64_t r1 = min(P.d, (int64_t)(it.tile0 + it.ntiles) * 128);
  double* o = reinterpret_cast<double*>(P.out) + (int64_t)it.col * P.ld;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) o[r] = 0.0;
}

// The columns the kernel marked NaN (it writes NaN to every row of a column holding a NaN / Inf; a
// column of finite values cannot produce a NaN) get the IEEE result: one warp per column, checked
// on row 0 of Â (n reads).
__global__ void sk_f4_ieee_fixup_kernel(const ApplyArgs P, const TcItem* items, int64_t n_items) {
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const double* out = reinterpret_cast<const double*>(P.out);
  for (int64_t i = warp0; i < n_items; i += nwarps) {
    const TcItem it = items[i];
    if (it.tile0 == 0 && it.pad != 2 && isnan(out[(int64_t)it.col * P.ld]))   // one item per column
      rad_ieee_fix_column<double>(P, it.col);
  }
}

cudaError_t launch_apply_rad_f4(const ApplyArgs& a, const TcItem* items, int64_t n_items, int64_t split_begin,
                                bool persist, cudaStream_t stream) {
  if (n_items == 0) return cudaSuccess;
  const size_t smem = (size_t)kF4Stages * kF4Stage + sizeof(F4Shared) + 1024;
  cudaError_t e = set_max_dynamic_smem((const void*)sk_rad_f4_kernel, smem);
  if (e != cudaSuccess) return e;
  static const int dbg = [] { const char* v = getenv("SKETCH_F4_DEBUG"); return v ? atoi(v) : 0; }();
  if (split_begin < n_items) {
    sk_f4_zero_split_kernel<<<(unsigned)(n_items - split_begin), 256, 0, stream>>>(a, items + split_begin);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && persist) {
    const size_t psmem = (size_t)kF4Stages * kF4PStage + sizeof(F4PShared) + 1024;
    e = set_max_dynamic_smem((const void*)sk_rad_f4p_kernel, psmem);
    int dev = 0, sms = 148;
    if (e == cudaSuccess) e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static const int grid_cap = [] { const char* v = getenv("SKETCH_F4_PGRID"); return v ? atoi(v) : 0; }();
    if (grid_cap > 0 && grid_cap < sms) sms = grid_cap;   // (tests: many items per CTA on small inputs)
    unsigned long long* ctr = nullptr;
    if (e == cudaSuccess) e = scratch_alloc((void**)&ctr, sizeof(unsigned long long), stream);
    if (e == cudaSuccess) {
      e = cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), stream);
      const int64_t grid = n_items < sms ? n_items : sms;
      if (e == cudaSuccess) {
        sk_rad_f4p_kernel<<<(unsigned)grid, kF4PThreads, psmem, stream>>>(a, items, n_items, ctr);
        e = cudaGetLastError();
      }
      const cudaError_t e2 = cudaFreeAsync(ctr, stream);
      if (e == cudaSuccess) e = e2;
    }
  } else if (e == cudaSuccess) {
    sk_rad_f4_kernel<<<(unsigned)n_items, kF4Threads, smem, stream>>>(a, items, dbg);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) {
    sk_f4_ieee_fixup_kernel<<<64, 256, 0, stream>>>(a, items, n_items);
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace sk
