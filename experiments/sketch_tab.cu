// sketch_tab.cu -- ±1 sketch of fp32 values through subset-sum tables (sm_100a).
//
// Per column k, Â[:, k] = Σ_p S[:, j_p] a_p (Algorithm 3's inner loops) with
// S = ±1 (bit 1 -> -1, include/sketch.h).  The SIMT kernel (sketch_kernels.cu) spends one
// predicated FADD per (row, nonzero) plus the predicate extraction.  Here the nonzero stream is
// cut into 32-nonzero chunks and each chunk into 8 groups of 4 nonzeros; for every group the CTA
// tabulates the 16 signed sums T_g[m] = Σ_{b<4} (bit b of m ? -a_{4g+b} : a_{4g+b}), and a row
// adds T_g[its 4 sign bits]: one LDS + one FADD per 4 (row, nonzero) entries.
//  * Warp w of the CTA owns Â rows 128 (tile0 + w) .. + 127 = Philox block q = tile0 + w.  Lane l
//    generates the block of nonzero l of the chunk; a 32 x 32 warp bit transpose (lane-rotated
//    words, 5 SHFL + LOP3 stages) leaves lane l with word qq = row 32 qq + l over the 32 nonzeros.
//  * Tables: 8 groups x 16 sums, each replicated for the 32 lanes ([g][m][lane], 16 KB per
//    chunk) so every LDS is conflict-free; built by all 512 threads, double-buffered, one
//    __syncthreads per chunk.  Sums are formed in nonzero order b = 0..3 (deterministic).
// Work item = (column, up to 16 row tiles of 128); fp32 accumulation like the SIMT kernel.
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.h"
#include "philox.cuh"

namespace sk {
namespace {

constexpr int kTbWarps = 16;
constexpr int kTbThreads = kTbWarps * 32;
constexpr int kTbTable = 8 * 16 * 32;             // floats per chunk: [group][sum index][lane]

// 32 x 32 bit transpose of 4 words across the warp (lane p word p in, lane r row r out), with
// words kept rotated left by the lane index so each stage is one SHFL + one LOP3.
__device__ __forceinline__ void tb_transpose(uint32_t (&x)[4], int lane) {
  const uint32_t m[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int k = 0; k < 4; ++k) x[k] = __funnelshift_l(x[k], x[k], lane);
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const uint32_t rm = __funnelshift_l(m[s], m[s], lane);
    const uint32_t keep = (lane & (16 >> s)) ? ~rm : rm;
    uint32_t y[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) y[k] = __shfl_xor_sync(0xFFFFFFFFu, x[k], 16 >> s);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(x[k]) : "r"(x[k]), "r"(y[k]), "r"(keep));
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) x[k] = __funnelshift_r(x[k], x[k], lane);
}

__global__ void __launch_bounds__(kTbThreads, 2) sk_rad_tab_kernel(const ApplyArgs P, const TcItem* items) {
  __shared__ __align__(16) float tab[2][kTbTable];
  const TcItem it = items[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t pb = P.colptr[it.col], pe = P.colptr[it.col + 1];
  const int64_t nch = (pe - pb + 31) >> 5;
  const bool active = warp < it.ntiles;
  const uint32_t q = (uint32_t)(it.tile0 + warp);
  const float* vals = reinterpret_cast<const float*>(P.vals);
  // table builder: thread i -> group tg, sum index tm, lanes 8 trq .. 8 trq + 7.  The values and
  // row indices of chunk c + 1 are loaded before chunk c is processed (global latency hidden).
  const int tg = threadIdx.x >> 6, tm = (threadIdx.x >> 2) & 15, trq = threadIdx.x & 3;
  auto load_a = [&](int64_t c, float (&a)[4]) {
    const int64_t p = pb + 32 * c + 4 * tg;
#pragma unroll
    for (int b = 0; b < 4; ++b) a[b] = p + b < pe ? __ldg(vals + p + b) : 0.0f;
  };
  auto load_j = [&](int64_t c) -> uint32_t {
    const int64_t p = pb + 32 * c + lane;
    return p < pe ? (uint32_t)__ldg(P.rowidx + p) : 0u;   // padding: a = 0 in the tables
  };
  auto store_table = [&](const float (&a)[4], float* T) {
    float s = 0.0f;
#pragma unroll
    for (int b = 0; b < 4; ++b) s += ((tm >> b) & 1) ? -a[b] : a[b];
    float4* dst = reinterpret_cast<float4*>(T + (tg * 16 + tm) * 32 + trq * 8);
    dst[0] = make_float4(s, s, s, s);
    dst[1] = make_float4(s, s, s, s);
  };
  float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  float an[4];
  uint32_t jc = 0;
  if (nch > 0) {
    load_a(0, an);
    store_table(an, tab[0]);
    jc = load_j(0);
  }
  __syncthreads();
  for (int64_t c = 0; c < nch; ++c) {
    const float* T = tab[c & 1] + lane;
    const bool more = c + 1 < nch;
    uint32_t jn = 0;
    if (more) { load_a(c + 1, an); jn = load_j(c + 1); }
    if (active) {
      const uint4 xb = s_block(q, (uint64_t)P.row_offset + jc, P.keys);
      uint32_t x[4] = {xb.x, xb.y, xb.z, xb.w};
      tb_transpose(x, lane);                       // word qq: row 32 qq + lane, bit k = nonzero k
#pragma unroll
      for (int qq = 0; qq < 4; ++qq)
#pragma unroll
        for (int g = 0; g < 8; ++g) acc[qq] += T[(g * 16 + ((x[qq] >> (4 * g)) & 15u)) * 32];
    }
    if (more) store_table(an, tab[(c + 1) & 1]);
    jc = jn;
    __syncthreads();
  }
  if (active) {
    float* outc = reinterpret_cast<float*>(P.out) + (int64_t)it.col * P.ld;
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
      const int64_t row = (int64_t)q * 128 + 32 * qq + lane;
      if (row < P.d) outc[row] = acc[qq];
    }
  }
}

}  // namespace

int tab_tiles_per_cta() { return kTbWarps; }

cudaError_t launch_apply_rad_tab(const ApplyArgs& a, const TcItem* items, int64_t n_items, cudaStream_t stream) {
  if (n_items == 0) return cudaSuccess;
  sk_rad_tab_kernel<<<(unsigned)n_items, kTbThreads, 0, stream>>>(a, items);
  return cudaGetLastError();
}

}  // namespace sk
