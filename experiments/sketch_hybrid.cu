// sketch_hybrid.cu -- ±1 sketch of fp64 values with the tensor cores AND the FP64 pipe busy at
// the same time, sm_100a.
//
// The two single-engine kernels are bounded by different units (profiles/r01_summary.md):
//  * the int8 tensor-core path (sk_rad_tc_kernel) is bounded by the tensor core's A-operand feed
//    (~46-62 (row, nonzero) entries/clk/SM) and needs only ~0.4 ALU ops per entry (Philox LOP3s +
//    one LOP3 per four S bytes);
//  * the SIMT path (sk_rad_kernel<double>) is bounded by the ALU pipe (one SEL per entry +
//    predicate generation, ~1.4 ALU ops per entry) and the FP64 pipe (one DADD per entry).
// One persistent CTA per SM runs both as warp-specialised groups that pull work items (column,
// up to 2048 rows of Â) from a single global queue ordered longest-first, so the split between
// the engines balances itself:
//   warps 0..3  : tensor-core producers (row tiles w, w+4, w+8, w+12: S tiles as {0,128} bytes,
//                 MN-major SWIZZLE_128B smem; value digits (8 int8 base-256 planes) by warp 0)
//                 + TMEM epilogue (warp w reads TMEM lane quarter w)
//   warp  4     : tcgen05.mma kind::i8 issuer (M=128, N=16, K=32 per row tile and K-step)
//   warps 5..12 : SIMT group, the sk_rad_kernel<double> algorithm with 8 warps
// (13 warps: at most 4 per scheduler, so every thread may use 128 registers.)
// Both engines are exact to the same bar as their standalone kernels.
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "kernels.h"
#include "philox.cuh"

namespace sk {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kHyTiles = 16;                      // 128-row tiles per item (2048 rows)
constexpr int kHyTcWarps = 4;                     // tensor-core producers (4 row tiles each)
constexpr int kHyMmaWarp = kHyTcWarps;            // warp 4
constexpr int kHySimtWarp0 = kHyTcWarps + 1;      // warps 5..12
constexpr int kHySimtWarps = 8;
constexpr int kHyThreads = (kHyTcWarps + 1 + kHySimtWarps) * 32;
constexpr int kHyStages = 2;
constexpr int kHyTile = 128 * 32;                 // A tile: M=128 x K=32 u8
constexpr int kHyStage = kHyTiles * kHyTile + 1024;
constexpr int kHyTmemCols = kHyTiles * 16;        // 16 int32 accumulators x N=16
constexpr int kHyXchWords = 5;
constexpr int kHyPad = 33;
constexpr int kHyRedBytes = kHySimtWarps * 32 * kHyPad * 8;   // 67.6 KB
constexpr int kHyXchBytes = kHySimtWarps * 32 * kHyXchWords * 4;

struct HyShared {
  uint64_t full[kHyStages];
  uint64_t empty[kHyStages];
  uint64_t done;          // MMAs of the current item finished (TC group)
  uint64_t tfree;         // epilogue finished reading TMEM (TC group)
  uint32_t tmem_base;
  int32_t tc_item;
  int32_t simt_item;
  int32_t E;
  int32_t nonfinite;
  int32_t T[8];
  unsigned long long maxabs_bits;
};

__device__ __forceinline__ uint32_t hs(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void hy_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(hs(b)), "r"(c));
}
__device__ __forceinline__ void hy_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(hs(b)) : "memory");
}
__device__ __forceinline__ void hy_wait(uint64_t* b, uint32_t parity) {
  asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
               "@!P1 bra WAIT_%=;\n\t}" :: "r"(hs(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void hy_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ uint64_t hy_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(layout & 7u) << 61;
  return d;
}
// kind::i8: D = S32, A = U8 MN-major, B = S8 MN-major, M = 128, N = 16
constexpr uint32_t kHyIdesc = (2u << 4) | (0u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | (2u << 17) | (8u << 24);

__device__ __forceinline__ int hy_row_of_m(int m) {   // M index -> row inside a 128-row tile
  const int blk = m >> 4, t = blk >> 1, h = blk & 1, u = (m >> 2) & 3, k = m & 3;
  return 32 * t + 8 * k + 4 * h + u;
}

// ---------------------------------------------------------------------------------------------
// SIMT group: sk_rad_kernel<double>'s algorithm with 8 warps over one item (column, <= 2048 rows).
__device__ void hy_simt_item(const ApplyArgs& P, const TcItem it, unsigned char* xch_base,
                             double* red, int w, int lane) {
  const int rows_item = it.ntiles * 128;
  const int WD = rows_item > 1024 ? 2 : 1;
  const int WK = kHySimtWarps / WD;
  const int wd = w % WD, wk = w / WD;
  const int64_t pb = P.colptr[it.col], pe = P.colptr[it.col + 1];
  const int64_t L = pe - pb;
  const int64_t s0 = pb + (L * wk) / WK, s1 = pb + (L * (wk + 1)) / WK;
  const int64_t row_base = (int64_t)it.tile0 * 128;
  const int64_t warp_row0 = row_base + (int64_t)wd * 1024;
  const uint32_t q = (uint32_t)(warp_row0 >> 7) + (uint32_t)(lane >> 2);
  const int t = lane & 3, g = lane >> 2;
  uint32_t* xch = reinterpret_cast<uint32_t*>(xch_base) + w * (32 * kHyXchWords);
  const double* vals = reinterpret_cast<const double*>(P.vals);
  double acc[32];
#pragma unroll
  for (int b = 0; b < 32; ++b) acc[b] = 0.0;
  for (int64_t p = s0; p < s1; p += 32) {
    const int cnt = (int)((s1 - p) < 32 ? (s1 - p) : 32);
    int32_t jl = 0;
    double al = 0.0;
    if (lane < cnt) { jl = __ldg(P.rowidx + p + lane); al = __ldg(vals + p + lane); }
    const int ngroups = (cnt + 3) >> 2;
    for (int u = 0; u < ngroups; ++u) {
      const uint32_t jr = (uint32_t)__shfl_sync(kFull, jl, 4 * u + t);
      const uint4 x = s_block(q, (uint64_t)P.row_offset + jr, P.keys);
      xch[lane * kHyXchWords + 0] = x.x;
      xch[lane * kHyXchWords + 1] = x.y;
      xch[lane * kHyXchWords + 2] = x.z;
      xch[lane * kHyXchWords + 3] = x.w;
      __syncwarp();
      uint32_t wv[4];
#pragma unroll
      for (int s = 0; s < 4; ++s) wv[s] = xch[(4 * g + s) * kHyXchWords + t];
      __syncwarp();
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const double a = __shfl_sync(kFull, al, 4 * u + s);
        const int lo = __double2loint(a), hi = __double2hiint(a), nhi = hi ^ (int)0x80000000;
#pragma unroll
        for (int b = 0; b < 32; ++b) {
          int h;
          asm("{.reg .pred p; .reg .b32 tt; and.b32 tt, %1, %4; setp.ne.u32 p, tt, 0; selp.b32 %0, %2, %3, p;}"
              : "=r"(h) : "r"(wv[s]), "r"(nhi), "r"(hi), "r"(1u << b));
          acc[b] += __hiloint2double(h, lo);
        }
      }
    }
  }
  double* mine = red + w * (32 * kHyPad) + lane * kHyPad;
#pragma unroll
  for (int b = 0; b < 32; ++b) mine[b] = acc[b];
  hy_bar(2, kHySimtWarps * 32);
  double* outc = reinterpret_cast<double*>(P.out) + (int64_t)it.col * P.ld;
  for (int r = w * 32 + lane; r < WD * 1024; r += kHySimtWarps * 32) {
    const int64_t row = row_base + r;
    if (row >= P.d || r >= rows_item) break;
    const int rwd = r >> 10, rr = r & 1023;
    const int off = (rr >> 5) * kHyPad + (rr & 31);
    double s = red[rwd * (32 * kHyPad) + off];
    for (int kk = 1; kk < WK; ++kk) s += red[(kk * WD + rwd) * (32 * kHyPad) + off];
    outc[row] = s;
  }
  hy_bar(2, kHySimtWarps * 32);   // red reusable
}

__global__ void __launch_bounds__(kHyThreads, 1)
sk_rad_hybrid_kernel(const ApplyArgs P, const TcItem* items, int n_items, int* counter, int mode) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* stages = smem_raw + ((1024u - (hs(smem_raw) & 1023u)) & 1023u);
  double* red = reinterpret_cast<double*>(stages + kHyStages * kHyStage);
  unsigned char* xch = stages + kHyStages * kHyStage + kHyRedBytes;
  HyShared& sh = *reinterpret_cast<HyShared*>(xch + kHyXchBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* vals = reinterpret_cast<const double*>(P.vals);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kHyStages; ++s) { hy_init(&sh.full[s], kHyTcWarps); hy_init(&sh.empty[s], 1); }
    hy_init(&sh.done, 1);
    hy_init(&sh.tfree, kHyTcWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kHyMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(hs(&sh.tmem_base)), "r"(kHyTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  const uint32_t tmem = sh.tmem_base;

  if (warp >= kHySimtWarp0) {
    // =============================== SIMT group ===============================
    const int w = warp - kHySimtWarp0;
    for (; mode != 1;) {
      if (w == 0 && lane == 0) sh.simt_item = atomicAdd(counter, 1);
      hy_bar(2, kHySimtWarps * 32);
      const int idx = sh.simt_item;
      hy_bar(2, kHySimtWarps * 32);
      if (idx >= n_items) break;
      hy_simt_item(P, items[idx], xch, red, w, lane);
    }
  } else {
    // =============================== tensor-core group ===============================
    // cumulative K-step count across items drives the stage-ring parities
    uint32_t gks = 0, nitem = 0;
    for (; mode != 2;) {
      if (warp == kHyMmaWarp && lane == 0) sh.tc_item = atomicAdd(counter, 1);
      hy_bar(1, (kHyTcWarps + 1) * 32);
      const int idx = sh.tc_item;
      if (warp < kHyTcWarps && threadIdx.x == 0) { sh.maxabs_bits = 0ull; sh.nonfinite = 0; }
      hy_bar(1, (kHyTcWarps + 1) * 32);
      if (idx >= n_items) break;
      const TcItem it = items[idx];
      const int64_t pb = P.colptr[it.col], pe = P.colptr[it.col + 1];
      const int nsteps = (int)((pe - pb + 31) >> 5);
      const int T = it.ntiles;
      if (warp < kHyTcWarps) {
        // ---- column scale E ----
        unsigned long long mx = col_absmax_bits(vals, pb, pe, threadIdx.x, kHyTcWarps * 32);
        for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, o));
        if (lane == 0) atomicMax(&sh.maxabs_bits, mx);
        hy_bar(3, kHyTcWarps * 32);
        if (threadIdx.x == 0) {
          const double m = __longlong_as_double((long long)sh.maxabs_bits);
          int e = 0;
          if (isfinite(m)) frexp(m, &e); else sh.nonfinite = 1;
          sh.E = e;
          for (int s = 0; s < 8; ++s) sh.T[s] = 0;
        }
        hy_bar(3, kHyTcWarps * 32);
        const int E = sh.E;
        const int e1 = 62 - E > 1000 ? 1000 : (62 - E < -1000 ? -1000 : 62 - E);
        const double sc1 = ldexp(1.0, e1), sc2 = ldexp(1.0, 62 - E - e1);
        // ---- producers: tiles warp + 4i; nonzero = lane ----
        int32_t Tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        auto load_j = [&](int ks) -> uint32_t {
          const int64_t p = pb + (int64_t)ks * 32 + lane;
          return (ks < nsteps && p < pe) ? (uint32_t)__ldg(P.rowidx + p) : 0u;
        };
        uint32_t j0 = load_j(0), j1 = load_j(1);
        double v0 = 0.0, v1 = 0.0;
        if (warp == 0) {
          const int64_t pa = pb + lane, pc = pb + 32 + lane;
          v0 = pa < pe ? __ldg(vals + pa) : 0.0;
          v1 = pc < pe ? __ldg(vals + pc) : 0.0;
        }
        for (int ks = 0; ks < nsteps; ++ks, ++gks) {
          const uint32_t j2 = load_j(ks + 2);
          double v2 = 0.0;
          if (warp == 0) { const int64_t pn = pb + (int64_t)(ks + 2) * 32 + lane; v2 = (ks + 2 < nsteps && pn < pe) ? __ldg(vals + pn) : 0.0; }
          const int stage = gks % kHyStages;
          const uint32_t use = gks / kHyStages;
          const int64_t p = pb + (int64_t)ks * 32 + lane;
          const bool live = p < pe;
          uint4 xs[4];
          const uint64_t J = (uint64_t)P.row_offset + j0;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            xs[i] = (live && warp + 4 * i < T) ? s_block((uint32_t)(it.tile0 + warp + 4 * i), J, P.keys)
                                               : make_uint4(0, 0, 0, 0);
          if (use > 0) hy_wait(&sh.empty[stage], (use - 1) & 1);
          unsigned char* st = stages + stage * kHyStage;
          const uint32_t sw = (uint32_t)(lane & 7);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int tt = warp + 4 * i;
            if (tt < T && live) {
              const uint32_t xw[4] = {xs[i].x, xs[i].y, xs[i].z, xs[i].w};
              const uint32_t base = hs(st + tt * kHyTile) + (uint32_t)(lane >> 3) * 1024u + sw * 128u;
#pragma unroll
              for (int tw = 0; tw < 4; ++tw) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                  uint32_t y[4];
#pragma unroll
                  for (int u = 0; u < 4; ++u) y[u] = (xw[tw] << (7 - (4 * h + u))) & 0x80808080u;
                  const uint32_t c = (uint32_t)(2 * tw + h);
                  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};"
                               :: "r"(base + ((c ^ sw) << 4)), "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]) : "memory");
                }
              }
            }
          }
          if (warp == 0) {
            uint32_t w0 = 0, w1 = 0;
            if (live) {
              long long A = __double2ll_rn((v0 * sc1) * sc2);
#pragma unroll
              for (int s = 0; s < 8; ++s) {
                const int c = (int)(signed char)(A & 0xFF);
                A = (A - c) >> 8;
                Tacc[s] += c;
                if (s < 4) w0 |= ((uint32_t)(c & 0xFF)) << (8 * s);
                else w1 |= ((uint32_t)(c & 0xFF)) << (8 * (s - 4));
              }
            }
            const uint32_t baddr = hs(st + kHyTiles * kHyTile) + (uint32_t)(lane >> 3) * 128u + (uint32_t)(lane & 7) * 16u;
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" :: "r"(baddr), "r"(w0), "r"(w1), "r"(0u), "r"(0u) : "memory");
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) hy_arrive(&sh.full[stage]);
          j0 = j1; j1 = j2;
          v0 = v1; v1 = v2;
        }
        if (warp == 0) {
#pragma unroll
          for (int s = 0; s < 8; ++s) {
            int v = Tacc[s];
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
            if (lane == 0) sh.T[s] = v;
          }
        }
        hy_bar(3, kHyTcWarps * 32);
        // ---- epilogue: warp w reads TMEM lane quarter w of every tile ----
        if (nsteps > 0) {
          hy_wait(&sh.done, nitem & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        const int qw = warp & 3;
        const int m = 32 * qw + lane;
        const int r = hy_row_of_m(m);
        double* outc = reinterpret_cast<double*>(P.out) + (int64_t)it.col * P.ld;
        const double nan = __longlong_as_double(0x7FF8000000000000ll);
        for (int tt = 0; tt < T; ++tt) {
          uint32_t D[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          if (nsteps > 0) {
            const uint32_t taddr = tmem + ((uint32_t)(32 * qw) << 16) + (uint32_t)(16 * tt);
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                         : "=r"(D[0]), "=r"(D[1]), "=r"(D[2]), "=r"(D[3]), "=r"(D[4]), "=r"(D[5]), "=r"(D[6]), "=r"(D[7])
                         : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
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
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) hy_arrive(&sh.tfree);
      } else {
        // ---- MMA issuer ----
        if (lane == 0) {
          if (nitem > 0) hy_wait(&sh.tfree, (nitem - 1) & 1);   // previous item's D has been read
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          uint32_t g = gks;
          for (int ks = 0; ks < nsteps; ++ks, ++g) {
            const int stage = g % kHyStages;
            hy_wait(&sh.full[stage], (g / kHyStages) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t sb = hs(stages + stage * kHyStage);
            const uint64_t bdesc = hy_desc(sb + kHyTiles * kHyTile, 128u, 128u, 0u);
            for (int tt = 0; tt < T; ++tt) {
              const uint64_t adesc = hy_desc(sb + tt * kHyTile, 4096u, 1024u, 2u);
              asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                           "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                           :: "r"(tmem + (uint32_t)(16 * tt)), "l"(adesc), "l"(bdesc), "r"(kHyIdesc),
                              "r"(ks > 0 ? 1u : 0u));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                         :: "r"(hs(&sh.empty[stage])) : "memory");
          }
          if (nsteps > 0)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                         :: "r"(hs(&sh.done)) : "memory");
          else
            hy_arrive(&sh.done);   // keep the done / tfree phases in step for empty items
        }
        __syncwarp();
        gks += nsteps;
      }
      ++nitem;
    }
  }
  __syncthreads();
  if (warp == kHyMmaWarp) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(kHyTmemCols));
  }
}

}  // namespace

int hybrid_tiles_per_item() { return kHyTiles; }

cudaError_t launch_apply_rad_hybrid(const ApplyArgs& a, const TcItem* items, int64_t n_items, int* counter,
                                    cudaStream_t stream) {
  if (n_items == 0) return cudaSuccess;
  const size_t smem = (size_t)kHyStages * kHyStage + kHyRedBytes + kHyXchBytes + sizeof(HyShared) + 1024;
  cudaError_t e = cudaFuncSetAttribute(sk_rad_hybrid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(counter, 0, sizeof(int), stream);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)(n_items < sms ? n_items : sms);
  // tuning knob: SKETCH_HYBRID_MODE = 1 (tensor-core group only) / 2 (SIMT group only)
  static const int mode = [] { const char* v = getenv("SKETCH_HYBRID_MODE"); return v ? atoi(v) : 0; }();
  sk_rad_hybrid_kernel<<<grid, kHyThreads, smem, stream>>>(a, items, (int)n_items, counter, mode);
  return cudaGetLastError();
}

}  // namespace sk
