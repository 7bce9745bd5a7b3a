// sketch_jki.cu -- Algorithm 4 ("jki"): one regeneration of S[:, j] per nonzero ROW
// of a column group, reused for every nonzero of that row in the group (uniform / Gaussian), sm_100a.
//
// Algorithm 3 (kji, sketch_kernels.cu) regenerates the column S[:, j] for every stored nonzero
// (j, k); Algorithm 4 walks A_sub row by row in CSR order ("A will need to be
// first partitioned into vertical blocks, and within each block, the entries will be stored in CSR
// format") and regenerates S[:, j] once per nonzero row j of the block.  On the GPU:
//  * vertical block = a group of kJCols = 16 consecutive columns of A; the plan (sketch_api.cu)
//    builds each group's CSR (distinct rows j, and per row its entries (column in group, index of the
//    value in the caller's CSC vals)) -- the paper's "format conversion", timed with the plan;
//  * work item = (group, tile of 1024 Â rows); warp w of the CTA owns rows row0 + 64 w .. + 63, lane l
//    rows 2l, 2l + 1 of those = the entries of ONE Philox block (q = row / 2);
//  * every warp walks the group's rows: one Philox block + transform per (row j, lane), then for each
//    entry (k, p) of row j: acc[k][2 rows] += S·vals[p], the warp's 64 x 16 accumulator tile in shared
//    memory (lane-contiguous, conflict-free), written to Â once at the end.
// RNG work is (nonzero rows of the group) x (d / 2) blocks instead of nnz x (d / 2): the reuse factor
// nnz / nnzrows per group (Abnormal_A of PAPER.md:697-707 -- dense rows -- reuses each block across
// all 16 columns).  For scattered sparsity the factor is ~1 and the plan keeps Algorithm 3.
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.h"
#include "philox.cuh"

namespace sk {
namespace {

constexpr int kJWarps = 16;
constexpr int kJRowsPerWarp = 64;
constexpr int kJRows = kJWarps * kJRowsPerWarp;   // Â rows per work item

template <int DIST, typename T>
__device__ __forceinline__ void jki_entries(const uint4 x, const double* __restrict__ logtab, T& v0, T& v1) {
  if constexpr (DIST == 1) {
    const double d0 = uniform53(x.x, x.y), d1 = uniform53(x.z, x.w);
    if constexpr (sizeof(T) == 8) { v0 = d0; v1 = d1; }
    else { v0 = __double2float_rn(d0); v1 = __double2float_rn(d1); }
  } else {
    double g0, g1;
    gaussian_pair_fast<kLogRep, 0>(x, logtab, nullptr, g0, g1);
    if constexpr (sizeof(T) == 8) { v0 = g0; v1 = g1; }
    else { v0 = __double2float_rn(g0); v1 = __double2float_rn(g1); }
  }
}

template <int DIST, typename T>
__global__ void __launch_bounds__(kJWarps * 32, 1) sk_jki_kernel(const ApplyArgs P, JkiPlanView J) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* acc = reinterpret_cast<T*>(smem);                                    // [warp][k][64 rows]
  double* logtab_base = reinterpret_cast<double*>(smem + kJWarps * kJCols * kJRowsPerWarp * sizeof(T));
  const double* logtab = logtab_base + (threadIdx.x & (kLogRep - 1));   // replicated -2 log table
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const JItem it = J.items[blockIdx.x];
  if constexpr (DIST == 2) {
    bm_fill_logtab(logtab_base);
  }
  T* mine = acc + warp * (kJCols * kJRowsPerWarp);
#pragma unroll
  for (int k = 0; k < kJCols; ++k) {
    mine[k * kJRowsPerWarp + 2 * lane] = T(0);
    mine[k * kJRowsPerWarp + 2 * lane + 1] = T(0);
  }
  __syncthreads();
  const int64_t row0 = (int64_t)it.row0 + (int64_t)warp * kJRowsPerWarp + 2 * lane;   // this lane's 2 rows
  const uint32_t q = (uint32_t)(row0 >> 1);
  const bool active = row0 < P.d;
  const T* vals = reinterpret_cast<const T*>(P.vals);
  const int64_t r_beg = J.grp_rows[it.group], r_end = J.grp_rows[it.group + 1];
  if (active) {
    for (int64_t r = r_beg; r < r_end; ++r) {
      const uint64_t j = (uint64_t)P.row_offset + (uint64_t)__ldg(J.row_j + r);
      const uint4 x = s_block(q, j, P.keys);
      T v0, v1;
      jki_entries<DIST, T>(x, logtab, v0, v1);
      const int64_t e_beg = __ldg(J.row_ent + r), e_end = __ldg(J.row_ent + r + 1);
      for (int64_t e = e_beg; e < e_end; ++e) {
        const uint32_t pk = __ldg(J.ent + e);                  // value index (bits 4..31) << 4 | column in group
        const int k = (int)(pk & (kJCols - 1));
        const T a = __ldg(vals + J.ent_base[it.group] + (pk >> 4));
        T* slot = mine + k * kJRowsPerWarp + 2 * lane;        // the lane's 2 rows, one vector access
        if constexpr (sizeof(T) == 8) {
          double2 c = *reinterpret_cast<double2*>(slot);
          c.x = fma(v0, a, c.x);
          c.y = fma(v1, a, c.y);
          *reinterpret_cast<double2*>(slot) = c;
        } else {
          float2 c = *reinterpret_cast<float2*>(slot);
          c.x = fmaf(v0, a, c.x);
          c.y = fmaf(v1, a, c.y);
          *reinterpret_cast<float2*>(slot) = c;
        }
      }
    }
  }
  __syncwarp();
  // one coalesced store per column of the group
  T* out = reinterpret_cast<T*>(P.out);
  const int64_t col0 = (int64_t)it.group * kJCols;
  for (int k = 0; k < kJCols; ++k) {
    const int64_t col = col0 + k;
    if (col >= J.n) break;
    T* outc = out + col * P.ld;
    if (row0 < P.d) outc[row0] = mine[k * kJRowsPerWarp + 2 * lane];
    if (row0 + 1 < P.d) outc[row0 + 1] = mine[k * kJRowsPerWarp + 2 * lane + 1];
  }
}

template <int DIST, typename T>
cudaError_t launch_jki_t(const ApplyArgs& a, const JkiPlanView& J, cudaStream_t stream) {
  const size_t smem = (size_t)kJWarps * kJCols * kJRowsPerWarp * sizeof(T) + (DIST == 2 ? kLogTabRepBytes : 0);
  cudaError_t e = cudaFuncSetAttribute(sk_jki_kernel<DIST, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  sk_jki_kernel<DIST, T><<<(unsigned)J.n_items, kJWarps * 32, smem, stream>>>(a, J);
  return cudaGetLastError();
}

}  // namespace

int jki_rows_per_item() { return kJRows; }

cudaError_t launch_apply_jki(int dist, int dtype, const ApplyArgs& a, const JkiPlanView& J, cudaStream_t stream) {
  if (J.n_items == 0) return cudaSuccess;
  if (dist == 1) return dtype == 0 ? launch_jki_t<1, double>(a, J, stream) : launch_jki_t<1, float>(a, J, stream);
  if (dist == 2) return dtype == 0 ? launch_jki_t<2, double>(a, J, stream) : launch_jki_t<2, float>(a, J, stream);
  return cudaErrorInvalidValue;
}

}  // namespace sk
