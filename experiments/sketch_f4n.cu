// sketch_f4n.cu -- ±1 sketch on the 5th-gen tensor cores, S as the N = 256 operand (sm_100a).
//
// Per column k, Â[:, k] = S[:, J_k] · a_k (Algorithm 3's inner loops) is a dense
// contraction over the column's nonzeros of a freshly generated ±1 matrix with the value vector.
// It runs EXACTLY on tcgen05.mma kind::mxf4 (block-scaled e2m1, f32 accumulation in TMEM):
//
//  * B operand = S tile, N = 256 Â rows x K = 64 nonzeros, K-major, packed e2m1: S[i, p] = ±1 is
//    the nibble 0x2 (+1.0) / 0xA (-1.0), the nibble's sign bit IS the Philox bit (bit 1 -> -1).
//  * A operand = the values as magnitude digits, M = 128 rows (64 used) x K = 64:
//    with e = frexp exponent of max_p |a_p| over the column (a separate pass, sk_colmax_kernel),
//    A_p = rint(a_p 2^(62-e)) (|A_p| <= 2^62; the rounding is the only approximation), and
//    A[s, p] = 2 sign(A_p) bit_s(|A_p|) in {0, ±2} (nibbles 0x0 / 0x4 / 0xC).  Padding nonzeros past
//    the column end have A_p = 0, so they contribute nothing whatever S holds.
//  * D[s, i] = Σ_p A[s, p] S[i, p] is an integer with |D| <= 2L < 2^24: exact in f32.
//    Â[i] = 2^(e-63) Σ_s 2^s D[s, i], formed from two exact fp64 partial sums and one rounding.
//    Error <= L 2^(e-63) <= 2^-62 L Σ_p |a_p|: below the 1e-12 bar; the fp64 partial sums
//    (|Σ_{s<32} 2^s D_s| < 2^32 2L) stay exact for L < 2^20 (kF4nMaxColumn).
//
// Why S is the N operand: an M = 128, K = 64 mxf4 MMA reads its A tile at ~44.5 B/clk/SM, so with
// S as A the tensor core consumes at most ~89 S entries/clk/SM; with S as B and N = 256 the MMA
// is compute-bound at ~128 clk for 16384 S entries (~128 entries/clk/SM, scripts/microbench_mxf4.cu).
//
// S producers: one Philox4x32-10 block (128 rows x 1 nonzero) per lane, then a 32 x 32 bit transpose
// across the warp so that lane r holds row r over 32 nonzeros (K-major).  The transpose uses
// lane-rotated words: lane l keeps its word rotated left by l, which turns every butterfly stage
// into SHFL + one LOP3 (no per-stage shift): 2 rotations + 5 LOP3 per word instead of 5 x (SHF +
// LOP3).  Nibble expansion ((y << (3-c)) & 0x88888888) | 0x22222222 puts nonzero 4n + c of the
// 32-nonzero half in nibble n of word c; the digits use the same transpose, so K orders agree.
//
// CTA (persistent, one per SM): NP S-producer warps + 2 digit warps + 1 loader warp (cp.async of
// rowidx / values into a K-step ring) + 1 MMA warp + 2 epilogue warps.  Work item = (column, 256-row
// tile of Â); a 3-stage smem ring of 4 K-steps each (A 4 KB + B 8 KB per K-step); accumulator
// D = TMEM columns [0, 256); scale factors (ue8m0 = 1.0) in columns [256, 320).  The epilogue dumps
// D to shared memory, releases the accumulator to the MMA warp for the next item, and then forms
// and stores Â while the next item's MMAs run.
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "philox.cuh"

namespace sk {
namespace {

constexpr int kNKS = 4;                           // K-steps (64 nonzeros) per smem stage
constexpr int kNStages = 3;
constexpr int kNCSlots = 8;                       // TMA ring of the nonzero stream, in chunks of kNKS K-steps
constexpr int kNChunk = 64 * kNKS;                // nonzeros per chunk (TMA box)
// A TMA box must start 16-byte aligned, so each chunk is loaded from its start rounded down to 4
// elements: a kNChunk box plus a 4-element tail box; consumers skip the first (start & 3).
constexpr int kNIdxBytes = 1152;                  // >= (kNChunk + 4) * 4, 128-byte multiple
constexpr int kNSlotBytes = kNIdxBytes + 2176;    // + (kNChunk + 4) * 8 values
constexpr int kNRows = 256;                       // Â rows per work item (MMA N)
constexpr int kNATile = 128 * 32;                 // digits: 128 rows x 64 fp4
constexpr int kNBTile = 256 * 32;                 // S: 256 rows x 64 fp4
constexpr int kNStage = kNKS * (kNATile + kNBTile);
constexpr int kNFStride = 33;                     // epilogue staging: digit pairs per Â row (+1 pad)
constexpr int kNFBytes = kNRows * kNFStride * 4;
constexpr uint32_t kNSfCol = 256;                 // TMEM scale-factor columns [256, 320)
#ifndef SK_SUSPEND_NS
#define SK_SUSPEND_NS 1000000
#endif
constexpr uint32_t kSuspendNs = SK_SUSPEND_NS;     // try_wait suspend-time hint (ns)

struct NShared {
  uint64_t full[kNStages];
  uint64_t empty[kNStages];
  uint64_t jfull[kNCSlots];
  uint64_t jempty[kNCSlots];
  uint64_t acc_full;
  uint64_t acc_free;
  uint32_t tmem_base;
};

constexpr size_t kNSmem = (size_t)kNStages * kNStage + (size_t)kNCSlots * kNSlotBytes + kNFBytes + sizeof(NShared) + 1024;

__device__ __forceinline__ uint32_t n_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void n_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(n_u32(bar)), "r"(count));
}
__device__ __forceinline__ void n_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(n_u32(bar)) : "memory");
}
// A macro so that ncu's source view attributes wait stalls to the call site.  N_SPIN selects a
// non-suspending test_wait poll loop instead of try_wait.
#ifndef N_SPIN
#define n_wait(bar, parity)                                                      \
  asm volatile(                                                                  \
      "{\n\t.reg .pred P1;\n\t"                                                  \
      "WAIT_%=:\n\t"                                                             \
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"               \
      "@!P1 bra WAIT_%=;\n\t}"                                                   \
      :: "r"(n_u32(bar)), "r"((uint32_t)(parity)), "r"(kSuspendNs) : "memory")
#else
#define n_wait(bar, parity)                                                      \
  asm volatile(                                                                  \
      "{\n\t.reg .pred P1;\n\t"                                                  \
      "WAIT_%=:\n\t"                                                             \
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"              \
      "@!P1 bra WAIT_%=;\n\t}"                                                   \
      :: "r"(n_u32(bar)), "r"((uint32_t)(parity)), "r"(0u) : "memory")
#endif

// Wait with back-off, for warps that idle for long stretches (epilogue, loader): frees issue slots.
__device__ __forceinline__ void n_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns) {
  uint32_t done;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(done) : "r"(n_u32(bar)), "r"(parity) : "memory");
    if (done) return;
    __nanosleep(ns);
  }
}

// K-major, no-swizzle smem descriptor: core matrix = 8 rows x 16 B; LBO = 128 B (next 16-byte K
// chunk), SBO = 256 B (next 8-row group); descriptor version 1 (sm_100).
__device__ __forceinline__ uint64_t n_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(256u >> 4) << 32) |
         ((uint64_t)1 << 46);
}

// kind::mxf4 instruction descriptor: A = B = E2M1, K-major, D = F32, scale E8M0, M = 128, N = 256.
__host__ __device__ constexpr uint32_t n_idesc() {
  return (1u << 7) | (1u << 10) | ((uint32_t)(kNRows >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);
}

// byte offset of row r, K half h inside a K-major no-swizzle tile
__device__ __forceinline__ uint32_t n_off(int r, int h) {
  return (uint32_t)((r >> 3) * 256 + h * 128 + (r & 7) * 16);
}

__device__ __forceinline__ uint32_t n_lop_sel(uint32_t x, uint32_t y, uint32_t k) {   // (x & k) | (y & ~k)
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(r) : "r"(x), "r"(y), "r"(k));
  return r;
}

// Per-lane stage masks of the rotated transpose: stage s (distance j = 16 >> s) keeps
// rot(m_j, lane) in the lower lane of a pair and its complement in the upper lane.
__device__ __forceinline__ void n_masks(uint32_t (&K)[5], int lane) {
  const uint32_t m[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const uint32_t r = __funnelshift_l(m[s], m[s], lane);
    K[s] = (lane & (16 >> s)) ? ~r : r;
  }
}

// 32 x 32 bit transpose of NW independent word sets across the warp: on entry lane p holds X[p]
// (bit b = row b, nonzero p), on exit lane r holds row r (bit c = nonzero c).  Words are kept
// rotated left by the lane index in between, so each stage is SHFL + LOP3.
template <int NW>
__device__ __forceinline__ void n_transpose(uint32_t (&x)[NW], int lane, const uint32_t (&K)[5]) {
#pragma unroll
  for (int k = 0; k < NW; ++k) x[k] = __funnelshift_l(x[k], x[k], lane);
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    uint32_t y[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) y[k] = __shfl_xor_sync(0xFFFFFFFFu, x[k], 16 >> s);
#pragma unroll
    for (int k = 0; k < NW; ++k) x[k] = n_lop_sel(x[k], y[k], K[s]);
  }
#pragma unroll
  for (int k = 0; k < NW; ++k) x[k] = __funnelshift_r(x[k], x[k], lane);
}

__device__ __forceinline__ uint32_t n_nib(uint32_t t) {   // (t & 0x88888888) | 0x22222222
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(t), "r"(0x88888888u), "r"(0x22222222u));
  return r;
}

// S row word y (bit c = nonzero c; 1 -> -1.0) -> 16 bytes of e2m1 nibbles; word c nibble n holds
// nonzero 4n + c.
__device__ __forceinline__ void n_store_s(uint32_t addr, uint32_t y) {
  const uint32_t w0 = n_nib(y << 3), w1 = n_nib(y << 2), w2 = n_nib(y << 1), w3 = n_nib(y);
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" :: "r"(addr), "r"(w0), "r"(w1), "r"(w2), "r"(w3) : "memory");
}

// Digit row word y (bit c = bit s of |A_c|) with sign word g (bit c = A_c < 0) -> nibbles
// 0x0 / 0x4 (+2.0) / 0xC (-2.0), same nonzero -> nibble map as n_store_s.
__device__ __forceinline__ uint32_t n_dig(uint32_t y, uint32_t g, int c) {
  const uint32_t t = y << (3 - c);                               // magnitude bit at nibble bit 3
  const uint32_t sg = (g << (3 - c)) & 0x88888888u;              // sign bit at nibble bit 3
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(t >> 1), "r"(0x44444444u), "r"(t & sg));   // (a & b) | c
  return r;
}
__device__ __forceinline__ void n_store_d(uint32_t addr, uint32_t y, uint32_t g) {
  const uint32_t w0 = n_dig(y, g, 0), w1 = n_dig(y, g, 1), w2 = n_dig(y, g, 2), w3 = n_dig(y, g, 3);
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" :: "r"(addr), "r"(w0), "r"(w1), "r"(w2), "r"(w3) : "memory");
}

template <typename T>
__device__ __forceinline__ double n_val(unsigned long long raw) {
  if constexpr (sizeof(T) == 8) return __longlong_as_double((long long)raw);
  else return (double)__uint_as_float((uint32_t)raw);
}

// max_p |a_p| per column as IEEE bits (non-negative doubles order like uint64; NaN > Inf > finite).
template <typename T>
__global__ void __launch_bounds__(256) sk_colmax_kernel(const int64_t* __restrict__ colptr, int64_t n,
                                                        const T* __restrict__ vals,
                                                        unsigned long long* __restrict__ colmax) {
  const int lane = threadIdx.x & 31;
  const int64_t base = colptr[0], nnz = colptr[n] - base;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t ch = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; ch * 1024 < nnz; ch += nw) {
    const int64_t p0 = base + ch * 1024, p1 = p0 + 1024 < base + nnz ? p0 + 1024 : base + nnz;
    int64_t p = p0 + lane;
    if (p >= p1) continue;
    int64_t lo = 0, hi = n;                        // largest c with colptr[c] <= p
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(colptr + mid) <= p) lo = mid; else hi = mid;
    }
    int64_t c = lo, cend = __ldg(colptr + c + 1);
    unsigned long long run = 0ull;
    for (; p < p1; p += 32) {
      while (p >= cend) {
        if (run) atomicMax(colmax + c, run);
        run = 0ull;
        ++c;
        cend = __ldg(colptr + c + 1);
      }
      const unsigned long long b = (unsigned long long)__double_as_longlong(fabs((double)__ldg(vals + p)));
      run = b > run ? b : run;
    }
    if (run) atomicMax(colmax + c, run);
  }
}

template <typename T, int NP>
__global__ void __launch_bounds__((NP + 8) * 32, 1)
sk_rad_f4n_kernel(const ApplyArgs P, const NItem* __restrict__ items, int64_t n_items,
                  const unsigned long long* __restrict__ colmax, const __grid_constant__ CUtensorMap tm_idx,
                  const __grid_constant__ CUtensorMap tm_idx4, const __grid_constant__ CUtensorMap tm_val,
                  const __grid_constant__ CUtensorMap tm_val4, int dbg) {
  constexpr int kUPW = 4 * kNKS / NP;             // S units (128 rows x 32 nonzeros) per warp per stage
  static_assert(kUPW * NP == 4 * kNKS, "NP must divide 4 * kNKS");
  // warps: S producers [0, NP), digit producers [NP, NP + 4) (one per scheduler), epilogue NP + 4, NP + 5
  // (TMEM lane quarters 0 and 1), TMA loader NP + 6, MMA NP + 7
  constexpr int wD0 = NP, wE0 = NP + 4, wL = NP + 6, wM = NP + 7;
  static_assert(wE0 % 4 == 0, "epilogue warps must own TMEM lane quarters 0 and 1");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* stages = smem_raw + ((1024u - (n_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* ring = stages + kNStages * kNStage;
  float* F = reinterpret_cast<float*>(ring + kNCSlots * kNSlotBytes);
  NShared& sh = *reinterpret_cast<NShared*>(reinterpret_cast<unsigned char*>(F) + kNFBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kNStages; ++s) { n_init(&sh.full[s], NP + 4); n_init(&sh.empty[s], 1); }
    for (int s = 0; s < kNCSlots; ++s) { n_init(&sh.jfull[s], 1); n_init(&sh.jempty[s], NP + 4); }
    n_init(&sh.acc_full, 1);
    n_init(&sh.acc_free, 2);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == wM) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(n_u32(&sh.tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // digit rows 64..127 of every A tile are zero for good
  for (int i = threadIdx.x; i < kNStages * kNKS * 64 * 2; i += blockDim.x) {
    const int t = i / 128, r = 64 + (i % 128) / 2, h = i & 1;
    const uint32_t a = n_u32(stages + (t / kNKS) * kNStage + (t % kNKS) * kNATile) + n_off(r, h);
    asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" :: "r"(a), "r"(0u) : "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const uint32_t tmem = sh.tmem_base;
  if (warp < 4) {   // scale factors = 1.0 (ue8m0 0x7F) in TMEM columns [256, 320), all 128 lanes
    const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + kNSfCol;
#pragma unroll
    for (int c = 0; c < 64; c += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};"
                   :: "r"(taddr + c), "r"(0x7F7F7F7Fu) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  __syncthreads();

  const int64_t d = P.d;
  uint32_t gc = 0, ga = 0;                        // global chunk and active-item counters
  if (warp < NP) {
    // ============================== S producers ==============================
    uint32_t K[5];
    n_masks(K, lane);
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
      const NItem I = items[it];
      const int nsteps = (I.L + 63) >> 6;
      const uint32_t qb = 2u * (uint32_t)I.tile;
      for (int c0 = 0; c0 < nsteps; c0 += kNKS, ++gc) {
        const int kcount = nsteps - c0 < kNKS ? nsteps - c0 : kNKS;
        const int stage = (int)(gc % kNStages);
        const uint32_t use = gc / kNStages;
        const int cs = (int)(gc % kNCSlots);
        const uint32_t* js = reinterpret_cast<const uint32_t*>(ring + cs * kNSlotBytes) + ((I.pb + 64 * c0) & 3);
        uint32_t x[4 * kUPW], jv[kUPW];
        n_wait(&sh.jfull[cs], (gc / kNCSlots) & 1);
#pragma unroll
        for (int i = 0; i < kUPW; ++i) {
          const int u = warp + NP * i;
          jv[i] = js[64 * (u >> 2) + 32 * (u & 1) + lane];   // past the column end: any row (digit 0)
        }
        __syncwarp();
        if (lane == 0) n_arrive(&sh.jempty[cs]);
#pragma unroll
        for (int i = 0; i < kUPW; ++i) {
          const int u = warp + NP * i;
          const uint4 b = s_block(qb + (uint32_t)((u >> 1) & 1), (uint64_t)P.row_offset + jv[i], P.keys);
          x[4 * i + 0] = b.x; x[4 * i + 1] = b.y; x[4 * i + 2] = b.z; x[4 * i + 3] = b.w;
        }
        if (!(dbg & 1)) n_transpose<4 * kUPW>(x, lane, K);
        if (use > 0) n_wait(&sh.empty[stage], (use - 1) & 1);
        const uint32_t sbase = n_u32(stages + stage * kNStage + kNKS * kNATile);
#pragma unroll
        for (int i = 0; i < kUPW; ++i) {
          const int u = warp + NP * i;
          if (u < 4 * kcount) {
            const uint32_t tile = sbase + (uint32_t)((u >> 2) * kNBTile);
            const int rb = (u >> 1) & 1, h = u & 1;
#pragma unroll
            for (int t = 0; t < 4; ++t) n_store_s(tile + n_off(128 * rb + 32 * t + lane, h), x[4 * i + t]);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) n_arrive(&sh.full[stage]);
      }
    }
  } else if (warp < wE0) {
    // ============================== digit producers (nonzero half h, K-steps kp, kp + 2) ==============================
    constexpr int kKD = kNKS / 2;
    const int h = (warp - wD0) & 1, kp = (warp - wD0) >> 1;
    uint32_t K[5];
    n_masks(K, lane);
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
      const NItem I = items[it];
      const int nsteps = (I.L + 63) >> 6;
      const double mx = __longlong_as_double((long long)colmax[I.col]);
      const bool fin = isfinite(mx);
      int e = 0;
      if (fin) frexp(mx, &e);
      // 2^(62-e) as two exact power-of-two factors
      const int e1 = 62 - e > 1000 ? 1000 : (62 - e < -1000 ? -1000 : 62 - e);
      const double sc1 = ldexp(1.0, e1), sc2 = ldexp(1.0, 62 - e - e1);
      for (int c0 = 0; c0 < nsteps; c0 += kNKS, ++gc) {
        const int kcount = nsteps - c0 < kNKS ? nsteps - c0 : kNKS;
        const int stage = (int)(gc % kNStages);
        const uint32_t use = gc / kNStages;
        const int cs = (int)(gc % kNCSlots);
        const T* vs = reinterpret_cast<const T*>(ring + cs * kNSlotBytes + kNIdxBytes) + ((I.pb + 64 * c0) & 3);
        uint32_t y[2 * kKD], sg[kKD];
        T v[kKD];
        n_wait(&sh.jfull[cs], (gc / kNCSlots) & 1);
#pragma unroll
        for (int q = 0; q < kKD; ++q) v[q] = vs[64 * (kp + 2 * q) + 32 * h + lane];
        __syncwarp();
        if (lane == 0) n_arrive(&sh.jempty[cs]);
#pragma unroll
        for (int q = 0; q < kKD; ++q) {
          // positions past the column end hold the next column's values: digit 0
          const bool inside = 64 * (c0 + kp + 2 * q) + 32 * h + lane < I.L;
          const long long A = (fin && inside) ? __double2ll_rn(((double)v[q] * sc1) * sc2) : 0ll;
          const bool neg = A < 0;
          const unsigned long long mag = (unsigned long long)(neg ? -A : A);
          sg[q] = __ballot_sync(0xFFFFFFFFu, neg);
          y[2 * q] = (uint32_t)mag;
          y[2 * q + 1] = (uint32_t)(mag >> 32);
        }
        n_transpose<2 * kKD>(y, lane, K);         // lane s: digit s (and 32 + s) over 32 nonzeros
        if (use > 0) n_wait(&sh.empty[stage], (use - 1) & 1);
        const uint32_t abase = n_u32(stages + stage * kNStage);
#pragma unroll
        for (int q = 0; q < kKD; ++q) {
          const int ks = kp + 2 * q;
          if (ks < kcount) {
            const uint32_t tile = abase + (uint32_t)(ks * kNATile);
            n_store_d(tile + n_off(lane, h), y[2 * q], sg[q]);
            n_store_d(tile + n_off(32 + lane, h), y[2 * q + 1], sg[q]);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) n_arrive(&sh.full[stage]);
      }
    }
  } else if (warp == wL) {
    // ============================== TMA loader: one chunk of rowidx + values per slot ==============================
    if (lane == 0) {
      constexpr uint32_t kBytes = (kNChunk + 4) * (4 + (uint32_t)sizeof(T));
      auto tma = [&](uint32_t dst, const CUtensorMap* m, int32_t coord, uint32_t bar) {
        asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                     :: "r"(dst), "l"(reinterpret_cast<uint64_t>(m)), "r"(coord), "r"(bar) : "memory");
      };
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        const NItem I = items[it];
        const int nsteps = (I.L + 63) >> 6;
        for (int c0 = 0; c0 < nsteps; c0 += kNKS, ++gc) {
          const int cs = (int)(gc % kNCSlots);
          const uint32_t use = gc / kNCSlots;
          if (use > 0) n_wait(&sh.jempty[cs], (use - 1) & 1);
          const uint32_t bar = n_u32(&sh.jfull[cs]);
          if (dbg & 8192) { n_arrive(&sh.jfull[cs]); continue; }
          const uint32_t dst = n_u32(ring + cs * kNSlotBytes);
          const int32_t coord = (int32_t)((I.pb + 64 * c0) & ~int64_t(3));
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(kBytes) : "memory");
          tma(dst, &tm_idx, coord, bar);
          tma(dst + 4 * kNChunk, &tm_idx4, coord + kNChunk, bar);
          tma(dst + kNIdxBytes, &tm_val, coord, bar);
          tma(dst + kNIdxBytes + (uint32_t)sizeof(T) * kNChunk, &tm_val4, coord + kNChunk, bar);
        }
      }
    }
    __syncwarp();
  } else if (warp == wM) {
    // ============================== MMA issuer ==============================
    if (lane == 0) {
      constexpr uint32_t idesc = n_idesc();
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        const NItem I = items[it];
        const int nsteps = (I.L + 63) >> 6;
        if (nsteps == 0) continue;
        if (ga > 0) n_wait(&sh.acc_free, (ga - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int c0 = 0; c0 < nsteps; c0 += kNKS, ++gc) {
          const int kcount = nsteps - c0 < kNKS ? nsteps - c0 : kNKS;
          const int stage = (int)(gc % kNStages);
          n_wait(&sh.full[stage], (gc / kNStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sb = n_u32(stages + stage * kNStage);
          for (int ks = 0; ks < kcount && !(dbg & 4); ++ks) {
            const uint64_t adesc = n_desc(sb + ks * kNATile);
            const uint64_t bdesc = n_desc(sb + kNKS * kNATile + ks * kNBTile);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}"
                :: "r"(tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"((c0 + ks) > 0 ? 1u : 0u),
                   "r"(tmem + kNSfCol), "r"(tmem + kNSfCol + 32u));
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                       :: "r"(n_u32(&sh.empty[stage])) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     :: "r"(n_u32(&sh.acc_full)) : "memory");
        ++ga;
      }
    }
    __syncwarp();
  } else {
    // ============================== epilogue (TMEM lane quarter qq: digits 32qq .. 32qq+31) ==============================
    const int qq = warp - wE0;
    const int t2 = 32 * qq + lane;
    const bool odd = lane & 1;
    T* out = reinterpret_cast<T*>(P.out);
    for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
      const NItem I = items[it];
      const int64_t r0 = (int64_t)I.tile * kNRows;
      T* outc = out + (int64_t)I.col * P.ld + r0;
      if (I.L == 0) {
        for (int r = t2; r < kNRows; r += 64)
          if (r0 + r < d) outc[r] = T(0);
        continue;
      }
      n_wait_sleep(&sh.acc_full, ga & 1, 128);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tb = tmem + ((uint32_t)(32 * qq) << 16);
#pragma unroll 1
      for (int c = 0; c < kNRows / 32; ++c) {
        uint32_t v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(tb + (uint32_t)(32 * c)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // digit pair (2p, 2p+1) -> D_2p + 2 D_2p+1 (exact in f32: |.| < 3 * 2^21); the even lane keeps
        // Â rows 0..15 of the 32, the odd lane rows 16..31
        float* f = F + (32 * c + (odd ? 16 : 0)) * kNFStride + (t2 >> 1);
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float mine = __uint_as_float(odd ? v[16 + k] : v[k]);
          const float other = __shfl_xor_sync(0xFFFFFFFFu, __uint_as_float(odd ? v[k] : v[16 + k]), 1);
          f[k * kNFStride] = odd ? fmaf(2.0f, mine, other) : fmaf(2.0f, other, mine);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) n_arrive(&sh.acc_free);      // the MMA warp may overwrite D now
      ++ga;
      asm volatile("bar.sync 1, 64;" ::: "memory");
      const double mx = __longlong_as_double((long long)colmax[I.col]);
      int e = 0;
      const bool fin = isfinite(mx);
      if (fin) frexp(mx, &e);
#pragma unroll 1
      for (int r = t2; r < kNRows; r += 64) {
        const float* f = F + r * kNFStride;
        double lo = 0.0, hi = 0.0, w = 1.0;
#pragma unroll
        for (int p = 0; p < 16; ++p) {            // exact: integers below 2^53
          lo = fma((double)f[p], w, lo);
          hi = fma((double)f[16 + p], w, hi);
          w *= 4.0;
        }
        const double val = scalbn(fma(hi, 4294967296.0, lo), e - 63);
        if (r0 + r < d) outc[r] = fin ? (T)val : (T)__longlong_as_double(0x7FF8000000000000ll);
      }
      asm volatile("bar.sync 1, 64;" ::: "memory");
    }
  }

  __syncthreads();
  if (warp == wM) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(512));
  }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link dependency).
PFN_cuTensorMapEncodeTiled_v12000 n_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// 1-D tiled tensor map over `count` elements with a box of kNChunk elements (OOB -> zero fill).
cudaError_t n_tensor_map(CUtensorMap* m, const void* base, CUtensorMapDataType type, uint64_t count, uint64_t esize,
                         uint32_t boxlen) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = n_encode_fn();
  if (!enc) return cudaErrorNotSupported;
  const cuuint64_t dim[1] = {count > 0 ? count : 1};
  const cuuint64_t stride[1] = {esize};            // rank 1: the driver still wants the array
  const cuuint32_t box[1] = {boxlen};
  const cuuint32_t es[1] = {1};
  const CUresult r = enc(m, type, 1, const_cast<void*>(base), dim, stride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <typename T, int NP>
cudaError_t launch_f4n_t(const ApplyArgs& a, const NItem* items, int64_t n_items, int64_t n_cols, int64_t nnz_end,
                         cudaStream_t stream) {
  CUtensorMap tm_idx, tm_idx4, tm_val, tm_val4;
  const CUtensorMapDataType vt = sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  cudaError_t e = n_tensor_map(&tm_idx, a.rowidx, CU_TENSOR_MAP_DATA_TYPE_INT32, (uint64_t)nnz_end, 4, kNChunk);
  if (e == cudaSuccess) e = n_tensor_map(&tm_idx4, a.rowidx, CU_TENSOR_MAP_DATA_TYPE_INT32, (uint64_t)nnz_end, 4, 4);
  if (e == cudaSuccess) e = n_tensor_map(&tm_val, a.vals, vt, (uint64_t)nnz_end, sizeof(T), kNChunk);
  if (e == cudaSuccess) e = n_tensor_map(&tm_val4, a.vals, vt, (uint64_t)nnz_end, sizeof(T), 4);
  if (e != cudaSuccess) return e;
  unsigned long long* colmax = nullptr;
  e = cudaMallocAsync((void**)&colmax, (size_t)(n_cols > 0 ? n_cols : 1) * 8, stream);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(colmax, 0, (size_t)(n_cols > 0 ? n_cols : 1) * 8, stream);
  if (e == cudaSuccess && n_cols > 0) {
    sk_colmax_kernel<T><<<148 * 8, 256, 0, stream>>>(a.colptr, n_cols, reinterpret_cast<const T*>(a.vals), colmax);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaFuncSetAttribute(sk_rad_f4n_kernel<T, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kNSmem);
  if (e == cudaSuccess) {
    int sms = 148;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t grid = n_items < sms ? n_items : sms;
    // dbg (tuning only; results invalid when nonzero): 1 = no S transposes, 4 = no MMAs
    static const int dbg = [] { const char* v = getenv("SKETCH_F4N_DEBUG"); return v ? atoi(v) : 0; }();
    sk_rad_f4n_kernel<T, NP><<<(unsigned)grid, (NP + 8) * 32, kNSmem, stream>>>(a, items, n_items, colmax, tm_idx,
                                                                                 tm_idx4, tm_val, tm_val4, dbg);
    e = cudaGetLastError();
  }
  cudaError_t e2 = cudaFreeAsync(colmax, stream);
  return e != cudaSuccess ? e : e2;
}

}  // namespace

bool f4n_aligned(const void* p) { return ((uintptr_t)p & 15u) == 0; }

cudaError_t launch_apply_rad_f4n(const ApplyArgs& a, int dtype, const NItem* items, int64_t n_items, int64_t n_cols,
                                 int64_t nnz_end, cudaStream_t stream) {
  if (n_items == 0) return cudaSuccess;
  static const int np = [] { const char* v = getenv("SKETCH_F4N_NP"); return v ? atoi(v) : 8; }();
  if (dtype == 0) return np == 16 ? launch_f4n_t<double, 16>(a, items, n_items, n_cols, nnz_end, stream)
                                  : launch_f4n_t<double, 8>(a, items, n_items, n_cols, nnz_end, stream);
  return np == 16 ? launch_f4n_t<float, 16>(a, items, n_items, n_cols, nnz_end, stream)
                  : launch_f4n_t<float, 8>(a, items, n_items, n_cols, nnz_end, stream);
}

}  // namespace sk
