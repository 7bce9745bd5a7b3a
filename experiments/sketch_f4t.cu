// sketch_f4t.cu -- ±1 sketch of fp64 values on the tensor cores with the S operand in TMEM (sm_100a).
//
// Same exact arithmetic as sketch_f4.cu (Algorithm 3's inner loops as a per-column
// contraction Â[:, k] = S[:, J_k] a_k): S = e2m1 ±1 nibbles (sign bit = Philox bit), values as 64
// signed binary digits of U_p = rint(a_p 2^(61-E)) + 2^63 plus an all-ones row, f32 accumulation of
// integers in TMEM, Â = 2^(E-62) (Σ_s 2^s D_s - D_64).  What changes is where S lives:
//
//  * sketch_f4.cu stages S in shared memory.  ncu shows its shared-memory data pipe ~80% busy
//    (STS of S 0.5 B/entry + tensor reads of S 0.5 B/entry + the transposes' SHFLs), which is what
//    binds it.  Here the producers write S straight into TMEM with tcgen05.st and the MMA reads its
//    A operand from TMEM (`tcgen05.mma ... [d], [a_tmem], b_desc`): an M=128 K=64 mxf4 MMA with A in
//    TMEM takes ~90 clk (scripts/microbench_mxf4.cu, layout 9), the same as from shared memory, and
//    shared memory now only carries the digits operand and the shuffles.
//  * A warp may only touch its own TMEM lane quarter (warp % 4).  Warp (quarter s, nonzero half h)
//    generates Philox block q0 + s (128 Â rows) for its 32 nonzeros; after the 32 x 32 transposes it
//    holds the rows of word t (rows 32t .. 32t+31 of that block) and stores them into lane quarter s
//    of MMA tile t.  MMA tile t therefore holds Â rows {128 s + 32 t + r : s = 0..3, r = 0..31} of the
//    item's 512 rows; the epilogue maps TMEM lane 32 s + r of tile t back to Â row 128 s + 32 t + r.
//  * TMEM: accumulators 4 tiles x 72 columns [0, 288), S buffers [288, 480) = 3 stages x 2 K-steps x
//    4 tiles x 8 columns (64 e2m1 per lane), scale factors (ue8m0 = 1.0) [480, 512).
// CTA = 8 S warps + 2 digit warps + 1 loader warp (cp.async ring of rowidx / values) + 1 MMA warp;
// one CTA per (column, 512-row block of Â).
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "kernels.h"
#include "philox.cuh"

namespace sk {
namespace {

constexpr int kTTiles = 4;                        // MMA tiles (M = 128) per item: 512 Â rows
#ifndef SK_F4T_SWARPS
#define SK_F4T_SWARPS 8
#endif
constexpr int kTSWarps = SK_F4T_SWARPS;           // S producers: (lane quarter s, nonzero half h, K-step class)
constexpr int kTKC = kTSWarps / 8;                // K-step classes: warp class c takes sub = c, c + kTKC, ...
constexpr int kTDWarps = 2;                       // digit producers: nonzero half
constexpr int kTProducers = kTSWarps + kTDWarps;
constexpr int kTLoaderWarp = kTProducers;
constexpr int kTMmaWarp = kTProducers + 1;
constexpr int kTThreads = (kTProducers + 2) * 32;
constexpr int kTSlots = 8;                        // nonzero-stream ring (K-steps of 64)
constexpr int kTN = 72;                           // 64 digit rows + ones row + 7 zero rows
#ifndef SK_F4T_SUB
#define SK_F4T_SUB 2
#define SK_F4T_STAGES 3
#endif
constexpr int kTSub = SK_F4T_SUB;                 // K-steps per stage
constexpr int kTStages = SK_F4T_STAGES;
constexpr int kTBSub = 2560;                      // digits tile (72 x 64 e2m1, padded) per K-step
constexpr int kTStage = kTSub * kTBSub;           // shared memory per stage (digits only)
constexpr uint32_t kTACol = kTTiles * kTN;        // S buffers start at TMEM column 288
constexpr uint32_t kTSfCol = 480;                 // scale factors: TMEM columns [480, 512)
static_assert(kTACol + kTStages * kTSub * kTTiles * 8 <= kTSfCol, "TMEM budget");

struct TShared {
  uint64_t full[kTStages];
  uint64_t empty[kTStages];
  uint64_t jfull[kTSlots];
  uint64_t jempty[kTSlots];
  uint64_t done;
  uint32_t js[kTSlots][64];
  double vs[kTSlots][64];
  uint32_t tmem_base;
  unsigned long long maxabs_bits;
  int32_t E;
  int32_t nonfinite;
};

__device__ __forceinline__ uint32_t t_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void t_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(t_u32(bar)), "r"(count));
}
__device__ __forceinline__ void t_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(t_u32(bar)) : "memory");
}
__device__ __forceinline__ void t_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}"
      :: "r"(t_u32(bar)), "r"(parity), "r"(1000000u) : "memory");
}

// K-major no-swizzle smem descriptor (digits operand): core matrix 8 rows x 16 B, LBO = 128 B,
// SBO = 256 B, version 1.
__device__ __forceinline__ uint64_t t_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(256u >> 4) << 32) |
         ((uint64_t)1 << 46);
}
// kind::mxf4 block-scaled: A = B = E2M1, K-major, D = F32, scale E8M0, M = 128, N = 72.
__host__ __device__ constexpr uint32_t t_idesc() {
  return (1u << 7) | (1u << 10) | ((uint32_t)(kTN >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);
}

// Lane-rotated 32 x 32 bit transposes (see sketch_f4.cu f4_transpose): lane p word p in, lane r row r out.
template <int NW>
__device__ __forceinline__ void t_transpose(uint32_t (&x)[NW], int lane) {
  const uint32_t m[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int k = 0; k < NW; ++k) x[k] = __funnelshift_l(x[k], x[k], lane);
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const uint32_t rm = __funnelshift_l(m[s], m[s], lane);
    const uint32_t keep = (lane & (16 >> s)) ? ~rm : rm;
    uint32_t y[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) y[k] = __shfl_xor_sync(0xFFFFFFFFu, x[k], 16 >> s);
#pragma unroll
    for (int k = 0; k < NW; ++k)
      asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(x[k]) : "r"(x[k]), "r"(y[k]), "r"(keep));
  }
#pragma unroll
  for (int k = 0; k < NW; ++k) x[k] = __funnelshift_r(x[k], x[k], lane);
}

__device__ __forceinline__ uint32_t t_nib(uint32_t t) {   // (t & 0x88888888) | 0x22222222
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(t), "r"(0x88888888u), "r"(0x22222222u));
  return r;
}
__device__ __forceinline__ uint32_t t_valid_mask(int c, int nvalid) {   // nibbles n with 4n + c < nvalid
  const int cnt = nvalid > c ? (nvalid - c + 3) >> 2 : 0;
  return cnt >= 8 ? 0xFFFFFFFFu : ((1u << (4 * cnt)) - 1u);
}
__device__ __forceinline__ uint32_t t_off(int m, int h) { return (uint32_t)((m >> 3) * 256 + h * 128 + (m & 7) * 16); }

// digits row word y -> 16 bytes of nibbles in shared memory, padding nonzeros (>= nvalid) = 0.0
__device__ __forceinline__ void t_store_digits(uint32_t addr, uint32_t y, int nvalid) {
  uint32_t w0 = t_nib(y << 3), w1 = t_nib(y << 2), w2 = t_nib(y << 1), w3 = t_nib(y);
  if (nvalid < 32) {
    w0 &= t_valid_mask(0, nvalid);
    w1 &= t_valid_mask(1, nvalid);
    w2 &= t_valid_mask(2, nvalid);
    w3 &= t_valid_mask(3, nvalid);
  }
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" :: "r"(addr), "r"(w0), "r"(w1), "r"(w2), "r"(w3) : "memory");
}

__global__ void __launch_bounds__(kTThreads, 1) sk_rad_f4t_kernel(const ApplyArgs P, const TcItem* items) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* stages = smem_raw + ((1024u - (t_u32(smem_raw) & 1023u)) & 1023u);
  TShared& sh = *reinterpret_cast<TShared*>(stages + kTStages * kTStage);
  const TcItem it = items[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t pb = P.colptr[it.col], pe = P.colptr[it.col + 1];
  const int64_t L = pe - pb;
  const int nsteps = (int)((L + 63) >> 6);
  const int nsup = (nsteps + kTSub - 1) / kTSub;
  const double* vals = reinterpret_cast<const double*>(P.vals);
  const uint32_t q0 = 4u * (uint32_t)it.tile0;    // first Philox block of the item's 512 rows

  if (threadIdx.x == 0) {
    for (int s = 0; s < kTStages; ++s) { t_init(&sh.full[s], kTProducers); t_init(&sh.empty[s], 1); }
    // a K-step slot is read by the S warps of one K-step class and by the digit warps
    for (int s = 0; s < kTSlots; ++s) { t_init(&sh.jfull[s], 32); t_init(&sh.jempty[s], kTSWarps / kTKC + kTDWarps); }
    t_init(&sh.done, 1);
    sh.maxabs_bits = 0ull;
    sh.nonfinite = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kTMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(t_u32(&sh.tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // digits rows 64..71 of every stage are constant: row 64 = +1.0 (0x2), rows 65..71 = 0
  for (int i = threadIdx.x; i < kTStages * kTSub * 8 * 2; i += blockDim.x) {
    const int s = i / (16 * kTSub), sub = (i / 16) % kTSub, row = 64 + (i % 16) / 2, h = i & 1;
    const uint32_t v = row == 64 ? 0x22222222u : 0u;
    const uint32_t a = t_u32(stages + s * kTStage + sub * kTBSub) + t_off(row, h);
    asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" :: "r"(a), "r"(v) : "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const uint32_t tmem = sh.tmem_base;
  if (warp < 4) {   // scale factors = 1.0 (ue8m0 0x7F) in TMEM columns [480, 512), all 128 lanes
    const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + kTSfCol;
#pragma unroll
    for (int c = 0; c < 32; c += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};"
                   :: "r"(taddr + c), "r"(0x7F7F7F7Fu) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  // column scale E (all producers)
  if (warp < kTProducers) {
    unsigned long long mx = col_absmax_bits(vals, pb, pe, threadIdx.x, kTProducers * 32);
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

  if (warp < kTSWarps) {
    // ===================== S producers: lane quarter s = warp % 4, nonzero half h =====================
    const int s = warp & 3, h = (warp >> 2) & 1, kc = warp >> 3;
    const uint32_t q = q0 + (uint32_t)s;
    const uint32_t tq = tmem + ((uint32_t)(32 * s) << 16);
    constexpr int kMine = kTSub / kTKC;          // K-steps of a stage this warp produces
    static_assert(kMine * kTKC == kTSub, "K-step classes must divide the stage");
    for (int ss = 0; ss < nsup; ++ss) {
      const int stage = ss % kTStages, use = ss / kTStages;
      uint32_t x[4 * kMine];
#pragma unroll
      for (int i = 0; i < kMine; ++i) {
        const int ks = kTSub * ss + kc + kTKC * i;
        uint32_t j = 0u;
        if (ks < nsteps) {
          const int slot = ks % kTSlots;
          t_wait(&sh.jfull[slot], (ks / kTSlots) & 1);
          j = sh.js[slot][32 * h + lane];
          __syncwarp();
          if (lane == 0) t_arrive(&sh.jempty[slot]);
        }
        const uint4 b = s_block(q, (uint64_t)P.row_offset + j, P.keys);   // padding nonzeros: digits 0
        x[4 * i + 0] = b.x; x[4 * i + 1] = b.y; x[4 * i + 2] = b.z; x[4 * i + 3] = b.w;
      }
      t_transpose<4 * kMine>(x, lane);            // lane r: row 32 t + r of block q over 32 nonzeros
      if (use > 0) t_wait(&sh.empty[stage], (use - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int i = 0; i < kMine; ++i) {
        const int sub = kc + kTKC * i;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const uint32_t y = x[4 * i + t];
          const uint32_t col = kTACol + (uint32_t)(((stage * kTSub + sub) * kTTiles + t) * 8 + 4 * h);
          asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};"
                       :: "r"(tq + col), "r"(t_nib(y << 3)), "r"(t_nib(y << 2)), "r"(t_nib(y << 1)), "r"(t_nib(y))
                       : "memory");
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) t_arrive(&sh.full[stage]);
    }
  } else if (warp < kTProducers) {
    // ===================== digit producers: nonzero half h =====================
    const int h = warp - kTSWarps;
    const int e1 = 61 - E > 1000 ? 1000 : (61 - E < -1000 ? -1000 : 61 - E);
    const double sc1 = ldexp(1.0, e1), sc2 = ldexp(1.0, 61 - E - e1);
    for (int ss = 0; ss < nsup; ++ss) {
      const int stage = ss % kTStages, use = ss / kTStages;
      uint32_t x[2 * kTSub];
      int nval[kTSub];
#pragma unroll
      for (int sub = 0; sub < kTSub; ++sub) {
        const int ks = kTSub * ss + sub;
        double v0 = 0.0;
        if (ks < nsteps) {
          const int slot = ks % kTSlots;
          t_wait(&sh.jfull[slot], (ks / kTSlots) & 1);
          v0 = sh.vs[slot][32 * h + lane];
          __syncwarp();
          if (lane == 0) t_arrive(&sh.jempty[slot]);
        }
        const int64_t c0 = pb + (int64_t)ks * 64 + 32 * h;
        nval[sub] = (int)(pe - c0 < 0 ? 0 : (pe - c0 > 32 ? 32 : pe - c0));
        // U = A + 2^63 (mod 2^64); digit s = +1 iff bit s of U; nibble sign = NOT bit
        unsigned long long U = 0ull;
        if (lane < nval[sub]) U = (unsigned long long)__double2ll_rn((v0 * sc1) * sc2) ^ 0x8000000000000000ull;
        x[2 * sub] = ~(uint32_t)U;
        x[2 * sub + 1] = ~(uint32_t)(U >> 32);
      }
      t_transpose<2 * kTSub>(x, lane);            // lane s: digit s (and 32 + s)
      if (use > 0) t_wait(&sh.empty[stage], (use - 1) & 1);
#pragma unroll
      for (int sub = 0; sub < kTSub; ++sub) {
        const uint32_t bt = t_u32(stages + stage * kTStage + sub * kTBSub);
        t_store_digits(bt + t_off(lane, h), x[2 * sub], nval[sub]);
        t_store_digits(bt + t_off(32 + lane, h), x[2 * sub + 1], nval[sub]);
        // the ones row: +1.0 for valid nonzeros, 0.0 for padding (rewritten every K-step)
        if (lane == 0) t_store_digits(bt + t_off(64, h), 0u, nval[sub]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) t_arrive(&sh.full[stage]);
    }
  } else if (warp == kTLoaderWarp) {
    // ===================== loader: rowidx / vals -> smem ring with cp.async ====================
    for (int ks = 0; ks < nsteps; ++ks) {
      const int slot = ks % kTSlots, use = ks / kTSlots;
      if (use > 0) t_wait(&sh.jempty[slot], (use - 1) & 1);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int64_t p = pb + (int64_t)ks * 64 + 32 * half + lane;
        const bool ok = p < pe;
        const int64_t ps = ok ? p : pb;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;"
                     :: "r"(t_u32(&sh.js[slot][32 * half + lane])), "l"(P.rowidx + ps), "r"(ok ? 4 : 0) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;"
                     :: "r"(t_u32(&sh.vs[slot][32 * half + lane])), "l"(vals + ps), "r"(ok ? 8 : 0) : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" :: "r"(t_u32(&sh.jfull[slot])) : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (warp == kTMmaWarp) {
    // ===================== MMA issuer: A (S) from TMEM, B (digits) from shared memory =====================
    if (lane == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      constexpr uint32_t idesc = t_idesc();
      for (int ss = 0; ss < nsup; ++ss) {
        const int stage = ss % kTStages;
        t_wait(&sh.full[stage], (ss / kTStages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int sub = 0; sub < kTSub; ++sub) {
          const int ks = kTSub * ss + sub;
          if (ks >= nsteps) break;
          const uint64_t bdesc = t_desc(t_u32(stages + stage * kTStage + sub * kTBSub));
#pragma unroll
          for (int t = 0; t < kTTiles; ++t) {
            const uint32_t acol = kTACol + (uint32_t)(((stage * kTSub + sub) * kTTiles + t) * 8);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%5], [%6], p;\n\t}"
                :: "r"(tmem + (uint32_t)(t * kTN)), "r"(tmem + acol), "l"(bdesc), "r"(idesc), "r"(ks > 0 ? 1u : 0u),
                   "r"(tmem + kTSfCol), "r"(tmem + kTSfCol + 8u));
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     :: "r"(t_u32(&sh.empty[stage])) : "memory");
      }
      if (nsteps > 0)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     :: "r"(t_u32(&sh.done)) : "memory");
    }
    __syncwarp();
  }

  // ===================== epilogue: S warps read D; warp (quarter s, g = warp / 4) takes tiles g, g + kTSWarps/4 ..
  if (warp < kTSWarps) {
    if (nsteps > 0) {
      t_wait(&sh.done, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    const int s = warp & 3, g = warp >> 2;
    double* outc = reinterpret_cast<double*>(P.out) + (int64_t)it.col * P.ld;
    const double nan = __longlong_as_double(0x7FF8000000000000ll);
    for (int t = g; t < kTTiles; t += kTSWarps / 4) {
      long long lo = 0, hi = 0, ones = 0;
      if (nsteps > 0) {
        const uint32_t base = tmem + ((uint32_t)(32 * s) << 16) + (uint32_t)(t * kTN);
#pragma unroll
        for (int c = 0; c < 72; c += 8) {
          uint32_t D[8];
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                       : "=r"(D[0]), "=r"(D[1]), "=r"(D[2]), "=r"(D[3]), "=r"(D[4]), "=r"(D[5]), "=r"(D[6]), "=r"(D[7])
                       : "r"(base + (uint32_t)c));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const long long dv = (long long)__float2ll_rn(__uint_as_float(D[u]));
            const int sd = c + u;
            if (sd < 32) lo += dv << sd;
            else if (sd < 64) hi += dv << (sd - 32);
            else if (sd == 64) ones = dv;
          }
        }
      }
      // TMEM lane 32 s + r of tile t holds Â row 128 s + 32 t + r of the item
      const int64_t row = (int64_t)it.tile0 * 512 + 128 * s + 32 * t + lane;
      if (row < P.d) {
        const double v = scalbn((double)hi * 4294967296.0 + (double)(lo - ones), E - 62);
        outc[row] = sh.nonfinite ? nan : v;
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  __syncthreads();
  if (warp == kTMmaWarp) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(512));
  }
}

}  // namespace

cudaError_t launch_apply_rad_f4t(const ApplyArgs& a, const TcItem* items, int64_t n_items, cudaStream_t stream) {
  if (n_items == 0) return cudaSuccess;
  // (at least 116 KB so that one CTA runs per SM: each CTA allocates all 512 TMEM columns)
  size_t smem = (size_t)kTStages * kTStage + sizeof(TShared) + 1024;
  if (smem < 116 * 1024) smem = 116 * 1024;
  cudaError_t e = cudaFuncSetAttribute(sk_rad_f4t_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  sk_rad_f4t_kernel<<<(unsigned)n_items, kTThreads, smem, stream>>>(a, items);
  return cudaGetLastError();
}

}  // namespace sk
