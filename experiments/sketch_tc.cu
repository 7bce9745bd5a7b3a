// sketch_tc.cu -- tcgen05 (5th-gen tensor core) path of the ±1 sketch for fp64 values, sm_100a.
//
// Per column k, Â[:, k] = S[:, J_k] · a_k is a dense contraction of a freshly generated
// d x L_k matrix with the column's value vector (Algorithm 3's inner loops).
// It runs on the tensor cores exactly (no rounding inside the contraction):
//
//  * values -> exact int8 digit planes.  With E = frexp-exponent of max_p |a_p| of the column,
//    A_p = rint(a_p 2^(62-E)) (|A_p| <= 2^62) is split into 8 balanced base-256 digits
//    c_{p,s} in [-128, 127], A_p = Σ_s c_{p,s} 256^s.  Rounding a_p to 2^(E-62) is the only
//    approximation: |error| <= L 2^(E-63) <= L 2^-62 Σ|a| (far below the 1e-12 |S||A| bar).
//  * signs -> bytes.  Â = T - 2P with T = Σ_p a_p and P_i = Σ_{p: bit(i,p)=1} a_p (the "T - 2P"
//    form of ±1).  The tensor core computes D_s[i] = Σ_p (128·bit(i,p)) · c_{p,s} with A = S-bytes
//    (u8, values {0, 128}) and B = digits (s8), accumulating exactly in int32 in TMEM
//    (|D| <= 2^14 L < 2^31 for L <= 131071, enforced by the plan).  The epilogue forms
//    Â[i] = Σ_s (T_s - D_s/64) 2^(8s+E-62) in fp64 (T_s = Σ_p c_{p,s}).
//  * S tiles are produced straight into shared memory in the MN-major (rows contiguous) int8
//    canonical layout: one Philox4x32-10 block = 128 bits = one 128-row column slice of S for one
//    nonzero = exactly one K index of a 128-row MMA tile.  Each lane expands its block with
//    IMAD.SHL + LOP3 ((x << (7-s)) & 0x80808080 -> four {0,128} bytes) and 8 STS.128.  Rows are
//    permuted inside the tile (M index m <-> row r(m) below) so the expansion needs no bit
//    gathering; the epilogue undoes the permutation.
//
// CTA = 16 producer warps (one 128-row tile each) + 1 MMA warp.  3-stage smem ring (A tiles
// 16 x 4 KB + B 512 B per stage = one K-step of 32 nonzeros), mbarrier full/empty handshake,
// tcgen05.mma kind::i8 M=128 N=16 K=32 (one per tile per K-step), tcgen05.commit releases the
// stage, TMEM holds 16 accumulators of 16 int32 columns.  Bound: shared-memory store bandwidth
// (1 byte of S per (row, nonzero)), ~2x the FP64 pipe roofline of the SIMT kernel.
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "kernels.h"
#include "philox.cuh"

namespace sk {
namespace {

constexpr int kTcTiles = 16;                 // 128-row tiles per CTA (max)
constexpr int kTcProducerWarps = kTcTiles;   // one producer warp per tile
constexpr int kTcThreads = (kTcProducerWarps + 1) * 32;
constexpr int kTcStages = 3;
constexpr int kTileBytes = 128 * 32;         // A tile: M=128 x K=32 int8
constexpr int kStageBytes = kTcTiles * kTileBytes + 1024;   // B tile padded: stages stay 1 KB aligned
constexpr int kTmemCols = kTcTiles * 16;     // 16 int32 accumulator columns per tile
constexpr uint32_t kMmaN = 16;

struct TcShared {
  uint64_t full[kTcStages];
  uint64_t empty[kTcStages];
  uint64_t done;
  uint32_t tmem_base;
  int32_t T[8];
  unsigned long long maxabs_bits;
  int32_t E;
  int32_t nonfinite;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t}"
      :: "r"(smem_u32(bar)), "r"(parity), "r"(0x989680u) : "memory");
}

// Canonical MN-major smem descriptors (Blackwell version 1).
//  * SWIZZLE_NONE: core matrices of 16 (MN) x 8 (K) bytes; SBO = stride between core matrices
//    along MN, LBO = stride between groups of 8 along K.  Used for the small B tile.
//  * SWIZZLE_128B: atoms of 128 bytes (MN) x 8 (K) rows, 16-byte chunk index XOR (row % 8);
//    LBO = stride between MN atoms, SBO = stride between K atoms.  Used for the S tiles: a
//    128-row tile is one atom wide, so one Philox block fills one swizzled 128-byte atom row
//    and both the producer stores and the tensor-core reads are bank-conflict free.
// layout: 0 = SWIZZLE_NONE, 2 = SWIZZLE_128B (atoms must be 1024-byte aligned).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;             // version = 1 (sm_100)
  d |= (uint64_t)(layout & 7u) << 61; // base_offset = 0, lbo_mode = 0
  return d;
}

// kind::i8 instruction descriptor: D = S32, A = U8 (MN-major), B = S8 (MN-major), M=128, N=16.
__host__ __device__ constexpr uint32_t make_idesc() {
  return (2u << 4)              // c_format = S32
       | (0u << 7)              // a_format = U8
       | (1u << 10)             // b_format = S8
       | (1u << 15)             // a_major = MN
       | (1u << 16)             // b_major = MN
       | ((kMmaN >> 3) << 17)   // n_dim
       | ((128u >> 4) << 24);   // m_dim
}

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
      :: "r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               :: "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(threads) : "memory");
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" :: "r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// Row (within a 128-row tile) held by MMA M index m: see the expansion in the producer loop.
__device__ __forceinline__ int tile_row_of_m(int m) {
  const int blk = m >> 4, t = blk >> 1, h = blk & 1, u = (m >> 2) & 3, k = m & 3;
  return 32 * t + 8 * k + 4 * h + u;
}

__global__ void __launch_bounds__(kTcThreads, 1) sk_rad_tc_kernel(const ApplyArgs P, const TcItem* items) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // carve: stages first (1 KB aligned for the 128-byte swizzle atoms), then bookkeeping
  unsigned char* stages = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  TcShared& sh = *reinterpret_cast<TcShared*>(stages + kTcStages * kStageBytes);
  const TcItem it = items[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t pb = P.colptr[it.col], pe = P.colptr[it.col + 1];
  const int64_t L = pe - pb;
  const int nsteps = (int)((L + 31) >> 5);
  const int ntiles = it.ntiles;
  const double* vals = reinterpret_cast<const double*>(P.vals);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; ++s) { mbar_init(&sh.full[s], kTcProducerWarps); mbar_init(&sh.empty[s], 1); }
    mbar_init(&sh.done, 1);
    sh.maxabs_bits = 0ull;
    sh.nonfinite = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kTcProducerWarps) {   // MMA warp owns the TMEM allocation
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(&sh.tmem_base)), "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();

  // ---- column scale: E = frexp exponent of max |a| (producers only) ----
  if (warp < kTcProducerWarps) {
    unsigned long long mx = col_absmax_bits(vals, pb, pe, threadIdx.x, kTcProducerWarps * 32);
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    if (lane == 0) atomicMax(&sh.maxabs_bits, mx);
    named_bar(1, kTcProducerWarps * 32);
    if (threadIdx.x == 0) {
      const double m = __longlong_as_double((long long)sh.maxabs_bits);
      int e = 0;
      if (isfinite(m)) frexp(m, &e); else sh.nonfinite = 1;
      sh.E = e;
      for (int s = 0; s < 8; ++s) sh.T[s] = 0;
    }
    named_bar(1, kTcProducerWarps * 32);
  }
  __syncthreads();
  const int E = sh.E;
  const uint32_t idesc = make_idesc();
  const uint32_t tmem_base = sh.tmem_base;

  if (warp < kTcProducerWarps) {
    // ======================= producers: S tiles (+ digits in warp 0) =======================
    const int t = warp;                                 // tile handled by this warp
    const bool has_tile = t < ntiles;
    const uint32_t q = (uint32_t)(it.tile0 + t);        // global 128-row tile = Philox block index
    int32_t Tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    // Software prefetch of the nonzero stream two K-steps ahead (rowidx for every warp, values
    // for warp 0), so the global-load latency overlaps the previous steps' generation.
    auto load_j = [&](int ks) -> uint32_t {
      const int64_t p = pb + (int64_t)ks * 32 + lane;
      return (ks < nsteps && p < pe) ? (uint32_t)__ldg(P.rowidx + p) : 0u;
    };
    auto load_v = [&](int ks) -> double {
      const int64_t p = pb + (int64_t)ks * 32 + lane;
      return (warp == 0 && ks < nsteps && p < pe) ? __ldg(vals + p) : 0.0;
    };
    uint32_t j0 = load_j(0), j1 = load_j(1);
    double v0 = load_v(0), v1 = load_v(1);
    for (int ks = 0; ks < nsteps; ++ks) {
      const uint32_t j2 = load_j(ks + 2);
      const double v2 = load_v(ks + 2);
      const int stage = ks % kTcStages;
      const int use = ks / kTcStages;
      if (use > 0) mbar_wait(&sh.empty[stage], (use - 1) & 1);
      unsigned char* st = stages + stage * kStageBytes;
      const int64_t p = pb + (int64_t)ks * 32 + lane;
      const bool live = p < pe;
      if (has_tile && live) {
        const uint64_t J = (uint64_t)P.row_offset + j0;
        const uint4 x = s_block(q, J, P.keys);
        const uint32_t xw[4] = {x.x, x.y, x.z, x.w};
        // K index = lane: K-atom lane/8 (1 KB), atom row lane%8 (128 B); the 16-byte chunk c
        // holding M indices 16c..16c+15 sits at physical chunk c ^ (lane % 8) (SWIZZLE_128B)
        const uint32_t base = smem_u32(st + t * kTileBytes) + (uint32_t)(lane >> 3) * 1024u + (uint32_t)(lane & 7) * 128u;
        const uint32_t sw = (uint32_t)(lane & 7);
#pragma unroll
        for (int tw = 0; tw < 4; ++tw) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t y[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int s = 4 * h + u;
              y[u] = (xw[tw] << (7 - s)) & 0x80808080u;   // bytes k: 128·bit(8k+s) of word tw
            }
            const uint32_t c = (uint32_t)(2 * tw + h);
            st_shared_v4(base + ((c ^ sw) << 4), y[0], y[1], y[2], y[3]);
          }
        }
      }
      if (warp == 0) {
        // B tile: digits of the 32 nonzeros (MN-major: 16 bytes per K index, N = 16, 8 used)
        uint32_t w0 = 0, w1 = 0;
        if (live) {
          long long A = __double2ll_rn(scalbn(v0, 62 - E));
#pragma unroll
          for (int s = 0; s < 8; ++s) {
            const int c = (int)(signed char)(A & 0xFF);
            A = (A - c) >> 8;
            Tacc[s] += c;
            if (s < 4) w0 |= ((uint32_t)(c & 0xFF)) << (8 * s);
            else w1 |= ((uint32_t)(c & 0xFF)) << (8 * (s - 4));
          }
        }
        const uint32_t baddr = smem_u32(st + kTcTiles * kTileBytes) + (uint32_t)(lane >> 3) * 128u + (uint32_t)(lane & 7) * 16u;
        st_shared_v4(baddr, w0, w1, 0u, 0u);
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.full[stage]);
      j0 = j1; j1 = j2;
      v0 = v1; v1 = v2;
    }
    if (warp == 0) {
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        int v = Tacc[s];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        if (lane == 0) sh.T[s] = v;
      }
    }
    named_bar(1, kTcProducerWarps * 32);

    // ======================= epilogue: TMEM -> fp64 -> Â =======================
    if (nsteps > 0) {
      mbar_wait(&sh.done, 0);
      fence_after();
    }
    const int quarter = warp & 3, group = warp >> 2;
    const int m = 32 * quarter + lane;
    const int r = tile_row_of_m(m);
    double* outc = reinterpret_cast<double*>(P.out) + (int64_t)it.col * P.ld;
    const double nan = __longlong_as_double(0x7FF8000000000000ll);
    for (int tt = group; tt < ntiles; tt += kTcProducerWarps / 4) {
      uint32_t D[16];
      if (nsteps > 0) {
        const uint32_t taddr = tmem_base + ((uint32_t)(32 * quarter) << 16) + (uint32_t)(16 * tt);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
            : "=r"(D[0]), "=r"(D[1]), "=r"(D[2]), "=r"(D[3]), "=r"(D[4]), "=r"(D[5]), "=r"(D[6]), "=r"(D[7]),
              "=r"(D[8]), "=r"(D[9]), "=r"(D[10]), "=r"(D[11]), "=r"(D[12]), "=r"(D[13]), "=r"(D[14]), "=r"(D[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      } else {
#pragma unroll
        for (int s = 0; s < 16; ++s) D[s] = 0;
      }
      const int64_t row = (int64_t)(it.tile0 + tt) * 128 + r;
      if (row < P.d) {
        double v = 0.0;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const double term = (double)sh.T[s] - (double)(int32_t)D[s] * 0.015625;
          v += scalbn(term, 8 * s + E - 62);
        }
        outc[row] = sh.nonfinite ? nan : v;
      }
    }
    fence_before();
  } else {
    // ======================= MMA issuer (one thread) =======================
    if (lane == 0) {
      for (int ks = 0; ks < nsteps; ++ks) {
        const int stage = ks % kTcStages;
        mbar_wait(&sh.full[stage], (ks / kTcStages) & 1);
        fence_after();
        const uint32_t sbase = smem_u32(stages + stage * kStageBytes);
        const uint64_t bdesc = make_desc(sbase + kTcTiles * kTileBytes, 128u, 128u, 0u);
        for (int tt = 0; tt < ntiles; ++tt) {
          const uint64_t adesc = make_desc(sbase + tt * kTileBytes, 4096u, 1024u, 2u);
          mma_i8(tmem_base + (uint32_t)(16 * tt), adesc, bdesc, idesc, ks > 0 ? 1u : 0u);
        }
        mma_commit(&sh.empty[stage]);
      }
      if (nsteps > 0) mma_commit(&sh.done);
    }
    __syncwarp();
  }
  __syncthreads();
  if (warp == kTcProducerWarps) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem_base), "r"(kTmemCols));
  }
}

// =============================================================================================
// Variant 2: S staged in TMEM (tcgen05.mma kind::i8 with A from TMEM, K-major).
//
// The tensor core reads an MN-major int8 A operand from shared memory at only ~62 B/clk/SM
// (scripts/microbench_umma.cu), which caps variant 1 at ~64 (row, nonzero) entries/clk/SM.  Here
// S never touches shared memory: every producer lane computes one Philox block (one nonzero x 128
// rows), the four 32-row words are exchanged through a small smem buffer (16 B per block), each
// warp transposes 32 x 32 bit blocks with 5 shuffle stages (lane r then holds row r's bits over
// the 32 nonzeros of the K-step), expands them to {0,128} bytes and writes its 32 TMEM lanes with
// tcgen05.st.  K order inside a K-step is permuted (K index kk <-> nonzero 8(kk%4) + kk/4) so the
// expansion is one shift + mask per 4 bytes; the B tile (digits) uses the same permutation.
// TMEM: columns [0, 256) = 16 accumulators (N = 16), [256, 512) = 2 stages x 16 A tiles x 8 cols.
constexpr int kTmStages = 2;
constexpr int kTmAccCols = kTcTiles * 16;
constexpr int kTmACols = kTcTiles * 8;               // one stage of A tiles (K = 32 bytes = 8 cols)
constexpr int kTmBlkBytes = kTcTiles * 4 * 32 * 4;   // [tile][word][lane] u32 = 8 KB per K-step
constexpr int kTmBBytes = 1024;                      // B tile (512 B used) per stage

struct TmShared {
  uint64_t full[kTmStages];
  uint64_t empty[kTmStages];
  uint64_t done;
  uint32_t tmem_base;
  int32_t T[8];
  unsigned long long maxabs_bits;
  int32_t E;
  int32_t nonfinite;
};

// kind::i8, D = S32, A = U8 K-major (TMEM), B = S8 MN-major (smem), M = 128, N = 16.
__host__ __device__ constexpr uint32_t make_idesc_ts() {
  return (2u << 4) | (0u << 7) | (1u << 10) | (0u << 15) | (1u << 16) | ((kMmaN >> 3) << 17) | ((128u >> 4) << 24);
}

__device__ __forceinline__ void mma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
      :: "r"(d_tmem), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// 32 x 32 bit-matrix transposes across the warp: on entry lane l holds word X[l] (bit b = entry
// (l, b)); on exit lane r holds bit l = X[l] bit r.  Stage j swaps the off-diagonal j x j blocks
// of every 2j x 2j block: one SHFL, one funnel rotate, one LOP3 per stage.
// Four independent transposes interleaved stage by stage (4 dependency chains for ILP).
__device__ __forceinline__ void transpose32x4(uint32_t (&x)[4], int lane) {
#pragma unroll
  for (int j = 16; j > 0; j >>= 1) {
    const uint32_t m = j == 16 ? 0x0000FFFFu : j == 8 ? 0x00FF00FFu : j == 4 ? 0x0F0F0F0Fu
                     : j == 2 ? 0x33333333u : 0x55555555u;
    const bool hi = (lane & j) != 0;
    const uint32_t keep = hi ? ~m : m;
    const uint32_t sh = hi ? (32 - j) : j;
    uint32_t y[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) y[k] = __shfl_xor_sync(0xFFFFFFFFu, x[k], j);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t t = __funnelshift_l(y[k], y[k], sh);
      x[k] = (x[k] & keep) | (t & ~keep);
    }
  }
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
               :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

__global__ void __launch_bounds__(kTcThreads, 1) sk_rad_tm_kernel(const ApplyArgs P, const TcItem* items) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint32_t* blk = reinterpret_cast<uint32_t*>(base);                         // 2 x 8 KB
  unsigned char* btiles = base + 2 * kTmBlkBytes;                            // kTmStages x 1 KB
  TmShared& sh = *reinterpret_cast<TmShared*>(btiles + kTmStages * kTmBBytes);
  const TcItem it = items[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t pb = P.colptr[it.col], pe = P.colptr[it.col + 1];
  const int64_t L = pe - pb;
  const int nsteps = (int)((L + 31) >> 5);
  const int ntiles = it.ntiles;
  const double* vals = reinterpret_cast<const double*>(P.vals);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmStages; ++s) { mbar_init(&sh.full[s], kTcProducerWarps); mbar_init(&sh.empty[s], 1); }
    mbar_init(&sh.done, 1);
    sh.maxabs_bits = 0ull;
    sh.nonfinite = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kTcProducerWarps) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(&sh.tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();

  if (warp < kTcProducerWarps) {
    unsigned long long mx = col_absmax_bits(vals, pb, pe, threadIdx.x, kTcProducerWarps * 32);
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    if (lane == 0) atomicMax(&sh.maxabs_bits, mx);
    named_bar(1, kTcProducerWarps * 32);
    if (threadIdx.x == 0) {
      const double m = __longlong_as_double((long long)sh.maxabs_bits);
      int e = 0;
      if (isfinite(m)) frexp(m, &e); else sh.nonfinite = 1;
      sh.E = e;
      for (int s = 0; s < 8; ++s) sh.T[s] = 0;
    }
    named_bar(1, kTcProducerWarps * 32);
  }
  __syncthreads();
  const int E = sh.E;
  const uint32_t tmem_base = sh.tmem_base;

  if (warp < kTcProducerWarps) {
    // Warp groups of 4: group g = warp / 4 owns tiles g, g+4, g+8, g+12.  Warp 4g+i generates
    // the Philox blocks of tile g+4i and writes TMEM lane quarter i of all four tiles, so the
    // block exchange only needs a 128-thread barrier inside the group.
    const int qw = warp & 3;
    const int g = warp >> 2;
    const int tp = g + 4 * qw;                     // tile whose blocks this warp generates
    const bool gen = tp < ntiles;
    const uint32_t q = (uint32_t)(it.tile0 + tp);
    const int kk_of_lane = 4 * (lane & 7) + (lane >> 3);   // K index of nonzero `lane`
    int32_t Tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    auto load_j = [&](int ks) -> uint32_t {
      const int64_t p = pb + (int64_t)ks * 32 + lane;
      return (ks < nsteps && p < pe) ? (uint32_t)__ldg(P.rowidx + p) : 0u;
    };
    uint32_t j0 = load_j(0), j1 = load_j(1);
    // values: this warp digitises K-steps ks = warp (mod 16); prefetch the next one
    double vnext = 0.0;
    {
      const int64_t p = pb + (int64_t)warp * 32 + lane;
      if (warp < nsteps && p < pe) vnext = __ldg(vals + p);
    }
    for (int ks = 0; ks < nsteps; ++ks) {
      const uint32_t j2 = load_j(ks + 2);
      const int stage = ks % kTmStages;
      const int use = ks / kTmStages;
      const int64_t p = pb + (int64_t)ks * 32 + lane;
      const bool live = p < pe;
      uint32_t* bb = blk + (ks & 1) * (kTmBlkBytes / 4);
      // 1) Philox block (tile tp, nonzero `lane`) -> [tile][word][lane]
      if (gen) {
        const uint4 x = live ? s_block(q, (uint64_t)P.row_offset + j0, P.keys) : make_uint4(0, 0, 0, 0);
        bb[(tp * 4 + 0) * 32 + lane] = x.x;
        bb[(tp * 4 + 1) * 32 + lane] = x.y;
        bb[(tp * 4 + 2) * 32 + lane] = x.z;
        bb[(tp * 4 + 3) * 32 + lane] = x.w;
      }
      named_bar(2 + g, 128);                     // the group's blocks are visible
      if (use > 0) mbar_wait(&sh.empty[stage], (use - 1) & 1);
      // 2) digits of this K-step's 32 nonzeros -> B tile (one warp per K-step, round robin)
      if ((ks & (kTcProducerWarps - 1)) == warp) {
        const double v0 = vnext;
        {
          const int64_t pn = pb + (int64_t)(ks + kTcProducerWarps) * 32 + lane;
          vnext = (ks + kTcProducerWarps < nsteps && pn < pe) ? __ldg(vals + pn) : 0.0;
        }
        uint32_t w0 = 0, w1 = 0;
        if (live) {
          long long A = __double2ll_rn(scalbn(v0, 62 - E));
#pragma unroll
          for (int s = 0; s < 8; ++s) {
            const int c = (int)(signed char)(A & 0xFF);
            A = (A - c) >> 8;
            Tacc[s] += c;
            if (s < 4) w0 |= ((uint32_t)(c & 0xFF)) << (8 * s);
            else w1 |= ((uint32_t)(c & 0xFF)) << (8 * (s - 4));
          }
        }
        const uint32_t baddr = smem_u32(btiles + stage * kTmBBytes) + (uint32_t)(kk_of_lane >> 3) * 128u +
                               (uint32_t)(kk_of_lane & 7) * 16u;
        st_shared_v4(baddr, w0, w1, 0u, 0u);
        fence_async_smem();
      }
      // 3) transpose + expand + TMEM store: quarter qw of tiles g, g+4, g+8, g+12
      uint32_t xw[4];
#pragma unroll
      for (int ii = 0; ii < 4; ++ii) {
        const int tt = g + 4 * ii;
        xw[ii] = tt < ntiles ? bb[(tt * 4 + qw) * 32 + lane] : 0u;
      }
      transpose32x4(xw, lane);                   // lane r: row 32qw + r over the 32 nonzeros
#pragma unroll
      for (int ii = 0; ii < 4; ++ii) {
        const int tt = g + 4 * ii;
        if (tt < ntiles) {
          uint32_t v[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) v[c] = (xw[ii] << (7 - c)) & 0x80808080u;   // byte b <- nonzero 8b + c
          const uint32_t taddr = tmem_base + ((uint32_t)(32 * qw) << 16) +
                                 (uint32_t)(kTmAccCols + stage * kTmACols + tt * 8);
          tmem_st8(taddr, v);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.full[stage]);
      j0 = j1; j1 = j2;
    }
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      int v = Tacc[s];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
      if (lane == 0 && v != 0) atomicAdd(&sh.T[s], v);
    }
    named_bar(1, kTcProducerWarps * 32);

    // ---- epilogue: D (lane m = tile row m) -> fp64 -> Â ----
    if (nsteps > 0) {
      mbar_wait(&sh.done, 0);
      fence_after();
    }
    const int m = 32 * qw + lane;
    double* outc = reinterpret_cast<double*>(P.out) + (int64_t)it.col * P.ld;
    const double nan = __longlong_as_double(0x7FF8000000000000ll);
    for (int tt = g; tt < ntiles; tt += 4) {
      uint32_t D[16];
      if (nsteps > 0) {
        const uint32_t taddr = tmem_base + ((uint32_t)(32 * qw) << 16) + (uint32_t)(16 * tt);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
            : "=r"(D[0]), "=r"(D[1]), "=r"(D[2]), "=r"(D[3]), "=r"(D[4]), "=r"(D[5]), "=r"(D[6]), "=r"(D[7]),
              "=r"(D[8]), "=r"(D[9]), "=r"(D[10]), "=r"(D[11]), "=r"(D[12]), "=r"(D[13]), "=r"(D[14]), "=r"(D[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      } else {
#pragma unroll
        for (int s = 0; s < 16; ++s) D[s] = 0;
      }
      const int64_t row = (int64_t)(it.tile0 + tt) * 128 + m;
      if (row < P.d) {
        double v = 0.0;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const double term = (double)sh.T[s] - (double)(int32_t)D[s] * 0.015625;
          v += scalbn(term, 8 * s + E - 62);
        }
        outc[row] = sh.nonfinite ? nan : v;
      }
    }
    fence_before();
  } else {
    if (lane == 0) {
      const uint32_t idesc = make_idesc_ts();
      for (int ks = 0; ks < nsteps; ++ks) {
        const int stage = ks % kTmStages;
        mbar_wait(&sh.full[stage], (ks / kTmStages) & 1);
        fence_after();
        const uint64_t bdesc = make_desc(smem_u32(btiles + stage * kTmBBytes), 128u, 128u, 0u);
        for (int tt = 0; tt < ntiles; ++tt) {
          const uint32_t a_tmem = tmem_base + (uint32_t)(kTmAccCols + stage * kTmACols + tt * 8);
          mma_i8_ts(tmem_base + (uint32_t)(16 * tt), a_tmem, bdesc, idesc, ks > 0 ? 1u : 0u);
        }
        mma_commit(&sh.empty[stage]);
      }
      if (nsteps > 0) mma_commit(&sh.done);
    }
    __syncwarp();
  }
  __syncthreads();
  if (warp == kTcProducerWarps) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem_base), "r"(512));
  }
}

}  // namespace

size_t tc_smem_bytes() { return (size_t)kTcStages * kStageBytes + sizeof(TcShared) + 1024; }
int tc_tiles_per_cta() { return kTcTiles; }

size_t tm_smem_bytes() { return (size_t)2 * kTmBlkBytes + kTmStages * kTmBBytes + sizeof(TmShared) + 1024; }

cudaError_t launch_apply_rad_tc(const ApplyArgs& a, const TcItem* items, int64_t n_items, int smem_staged,
                                cudaStream_t stream) {
  if (n_items == 0) return cudaSuccess;
  if (!smem_staged) {
    const size_t smem = tm_smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(sk_rad_tm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    sk_rad_tm_kernel<<<(unsigned)n_items, kTcThreads, smem, stream>>>(a, items);
    return cudaGetLastError();
  }
  const size_t smem = tc_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(sk_rad_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  sk_rad_tc_kernel<<<(unsigned)n_items, kTcThreads, smem, stream>>>(a, items);
  return cudaGetLastError();
}

}  // namespace sk
