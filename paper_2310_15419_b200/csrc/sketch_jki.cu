// sketch_jki.cu -- Algorithm 4 ("jki") with full row reuse: S[:, j] is regenerated
// ONCE per nonzero row j of a vertical block of up to b_n columns (b_n = all n when the block's
// accumulator fits in shared memory) and applied to every nonzero of that row (uniform / Gaussian),
// sm_100a.
//
// The paper's Algorithm 4 walks A row by row inside vertical blocks stored in CSR ("A will need to be
// first partitioned into vertical blocks, and within each block, the entries will be stored in CSR
// format") and says to "tune b_n to minimize the number of random variables
// generated": the RNG work is Σ_blocks nonzero rows x d instead of nnz x d.  With
// b_n = n every needed entry of S is generated exactly once (the strict count of SURVEY.md §8(d)).
// On the GPU:
//  * work item = (tile of kJRows = 16 rows of Â, block, range of the block's row batches): the CTA
//    keeps the 16 x b_n accumulator of its tile in shared memory (fp64: 128 B per column, b_n <= 1024);
//  * a batch = up to kJBatch = 128 nonzero rows (<= kJBatchEnt = 1024 entries).  Stage (all 512
//    threads): S[tile rows, j] for the batch's rows -- 1024 Philox blocks, two per thread -- into
//    shared memory, and the batch's entries (column, row slot, value);
//  * scatter: half-warp h (32 per CTA) owns the block's columns k = h mod 32 and applies the batch's
//    entries of its columns in row order, lane i updating row i: acc[k][i] += S[slot][i] a.  Entries
//    of one column are applied by one half-warp in a fixed order, so results are deterministic;
//  * latency: a first kernel gathers the values into the blocks' CSR order (vals_csr[e] = vals[p_e],
//    coalesced writes), so a batch's inputs are plain sequential loads, issued one batch ahead into
//    registers; S and the entries are double-buffered, so the scatter of batch b and the stage of
//    batch b+1 run between the same two barriers (one __syncthreads per batch) and one warp's
//    scatter latency hides under the other warps' Philox work;
//  * the tile's accumulator is written to Â once (or, when the block's batches are split over several
//    items for load balance, to a workspace slot that a finishing kernel sums in a fixed order).
// The plan (sketch_api.cu) builds the blocks' CSR on the host -- the paper's "format conversion",
// timed with the plan -- and only when the exact per-block distinct-row count makes it pay.
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.h"
#include "philox.cuh"

namespace sk {
namespace {

constexpr int kJThreads = 512;
constexpr int kJLogRep = 8;          // replicated -2 log table: 8 copies (24.8 KB)
constexpr int kJLogBytes = kBmLogRows * 3 * kJLogRep * 8;

template <typename T>
constexpr size_t jki_smem_bytes(int bn) {
  return (size_t)bn * kJRows * sizeof(T)                 // accumulator
         + 2 * (size_t)kJBatch * kJRows * sizeof(T)     // S of two batches
         + 2 * (size_t)kJBatchEnt * (4 + sizeof(T))     // entries (descriptor, value) of two batches
         + 2 * 64 * 2                                   // owner offsets of two batches (33 used)
         + kJLogBytes;
}

__device__ __forceinline__ void jki_fill_logtab(double* t) {
  for (int i = threadIdx.x; i < kBmLogRows * 3 * kJLogRep; i += blockDim.x) t[i] = (&kBmLogTab[0][0])[i / kJLogRep];
}

template <int DIST, typename T>
__device__ __forceinline__ void jki_entries(const uint4 x, const double* __restrict__ logtab, T& v0, T& v1) {
  if constexpr (DIST == 1) {
    const double d0 = uniform53(x.x, x.y), d1 = uniform53(x.z, x.w);
    if constexpr (sizeof(T) == 8) { v0 = d0; v1 = d1; }
    else { v0 = __double2float_rn(d0); v1 = __double2float_rn(d1); }
  } else {
    double g0, g1;
    gaussian_pair_fast<kJLogRep, 0>(x, logtab, nullptr, g0, g1);
    if constexpr (sizeof(T) == 8) { v0 = g0; v1 = g1; }
    else { v0 = __double2float_rn(g0); v1 = __double2float_rn(g1); }
  }
}

constexpr int kJSlotsPerThread = kJBatch * (kJRows / 2) / kJThreads;   // 2 Philox blocks per thread
constexpr int kJEntPerThread = kJBatchEnt / kJThreads;                  // 2 entries per thread

// One batch's inputs as one thread loads them (registers): its rows and its entries.
template <typename T>
struct JRegs {
  int32_t rj[kJSlotsPerThread];
  uint32_t desc[kJEntPerThread];
  T val[kJEntPerThread];
  uint16_t own;
  int nrows, nent;
};

template <typename T>
__device__ __forceinline__ void jki_load(const JkiPlanView& J, const T* __restrict__ vcsr, int64_t bt, JRegs<T>& R) {
  const JBatch B = J.batches[bt];
  R.nrows = B.nrows;
  R.nent = B.nent;
  const int tid = threadIdx.x;
#pragma unroll
  for (int h = 0; h < kJSlotsPerThread; ++h) {
    const int slot = (tid >> 3) + 64 * h;
    R.rj[h] = slot < B.nrows ? __ldg(J.row_j + B.row0 + slot) : 0;
  }
#pragma unroll
  for (int k = 0; k < kJEntPerThread; ++k) {
    const int e = tid + kJThreads * k;
    R.desc[k] = e < B.nent ? __ldg(J.ent_desc + B.ent0 + e) : 0u;
    R.val[k] = e < B.nent ? __ldg(vcsr + B.ent0 + e) : T(0);
  }
  R.own = tid < kJOwners + 1 ? __ldg(J.own + bt * (kJOwners + 1) + tid) : 0;
}

template <int DIST, typename T>
__global__ void __launch_bounds__(kJThreads, 1) sk_jki_kernel(const ApplyArgs P, const JkiPlanView J,
                                                               const T* __restrict__ vcsr, T* __restrict__ ws) {
  extern __shared__ __align__(16) unsigned char smem[];
  const JItem it = J.items[blockIdx.x];
  const int64_t c0 = (int64_t)it.block * J.bn;
  const int nbc = (int)min((int64_t)J.bn, J.n - c0);              // columns of this block
  T* acc = reinterpret_cast<T*>(smem);                             // [nbc][kJRows]
  T* S = acc + (size_t)J.bn * kJRows;                              // [2][kJBatch][kJRows]
  uint32_t* edesc = reinterpret_cast<uint32_t*>(S + 2 * kJBatch * kJRows);   // [2][kJBatchEnt]
  T* evals = reinterpret_cast<T*>(edesc + 2 * kJBatchEnt);         // [2][kJBatchEnt]
  uint16_t* own = reinterpret_cast<uint16_t*>(evals + 2 * kJBatchEnt);       // [2][64]
  double* logtab = reinterpret_cast<double*>(own + 2 * 64);
  const double* mylog = logtab + (threadIdx.x & (kJLogRep - 1));
  const int tid = threadIdx.x;
  const uint32_t q0 = (uint32_t)it.tile * (kJRows / 2);            // Philox block of the tile's first row
  const int ql = tid & 7;

  for (int e = tid; e < nbc * kJRows; e += kJThreads) acc[e] = T(0);
  if constexpr (DIST == 2) jki_fill_logtab(logtab);

  // stage: the batch held in R -> buffer b (S rows: 2 Philox blocks per thread; entries; owners)
  auto stage = [&](const JRegs<T>& R, int b) {
    T* Sb = S + b * (kJBatch * kJRows);
#pragma unroll
    for (int h = 0; h < kJSlotsPerThread; ++h) {
      const int slot = (tid >> 3) + 64 * h;
      if (slot < R.nrows) {
        const uint4 x = s_block(q0 + ql, (uint64_t)P.row_offset + (uint32_t)R.rj[h], P.keys);
        T v0, v1;
        jki_entries<DIST, T>(x, mylog, v0, v1);
        Sb[slot * kJRows + 2 * ql] = v0;
        Sb[slot * kJRows + 2 * ql + 1] = v1;
      }
    }
#pragma unroll
    for (int k = 0; k < kJEntPerThread; ++k) {
      const int e = tid + kJThreads * k;
      if (e < R.nent) { edesc[b * kJBatchEnt + e] = R.desc[k]; evals[b * kJBatchEnt + e] = R.val[k]; }
    }
    if (tid < kJOwners + 1) own[b * 64 + tid] = R.own;
  };

  JRegs<T> R;
  if (it.bt0 < it.bt1) {
    if constexpr (DIST == 2) __syncthreads();                      // the log table before the first stage
    jki_load(J, vcsr, it.bt0, R);
    stage(R, 0);
    if (it.bt0 + 1 < it.bt1) jki_load(J, vcsr, it.bt0 + 1, R);     // in flight during the first scatter
  }
  __syncthreads();
  const int hw = tid >> 4, i = tid & 15;                           // half-warp = column owner, lane = row
  for (int64_t bt = it.bt0; bt < it.bt1; ++bt) {
    const int b = (int)((bt - it.bt0) & 1);
    const T* Sb = S + b * (kJBatch * kJRows);
    const int e1 = own[b * 64 + hw + 1];
    for (int e = own[b * 64 + hw]; e < e1; ++e) {
      const uint32_t dsc = edesc[b * kJBatchEnt + e];
      T* slot = acc + (dsc & 0xFFFFu) * kJRows + i;
      *slot = fma(Sb[(dsc >> 16) * kJRows + i], evals[b * kJBatchEnt + e], *slot);
    }
    if (bt + 1 < it.bt1) {
      stage(R, b ^ 1);
      if (bt + 2 < it.bt1) jki_load(J, vcsr, bt + 2, R);           // in flight during the next scatter
    }
    __syncthreads();
  }

  // the tile's rows [16 tile, +16) of the block's columns: to Â, or to this item's workspace slot
  const int64_t row0 = (int64_t)it.tile * kJRows;
  T* dst = it.slot < 0 ? reinterpret_cast<T*>(P.out) + c0 * P.ld
                       : ws + (size_t)it.slot * (size_t)J.bn * (size_t)P.d;
  for (int e = tid; e < nbc * kJRows; e += kJThreads) {
    const int c = e >> 4, r = e & 15;
    if (row0 + r < P.d) dst[(int64_t)c * P.d + row0 + r] = acc[e];
  }
}

// The values in the blocks' CSR order (one coalesced pass; the kernel's entries are then sequential).
template <typename T>
__global__ void sk_jki_gather_kernel(const T* __restrict__ vals, const uint32_t* __restrict__ ent_p, int64_t n,
                                     T* __restrict__ vcsr) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    vcsr[e] = __ldg(vals + __ldg(ent_p + e));
}

// Blocks whose batches were split over several items: Â = Σ_parts in slot order (deterministic).
template <typename T>
__global__ void sk_jki_finish_kernel(const ApplyArgs P, const JkiPlanView J, const T* __restrict__ ws) {
  T* out = reinterpret_cast<T*>(P.out);
  for (int b = 0; b < J.n_blocks; ++b) {
    const int s0 = J.blk_slot[b], s1 = J.blk_slot[b + 1];
    if (s1 - s0 < 1) continue;
    const int64_t c0 = (int64_t)b * J.bn;
    const int64_t nel = min((int64_t)J.bn, J.n - c0) * P.d;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nel; e += (int64_t)gridDim.x * blockDim.x) {
      T s = ws[(size_t)s0 * J.bn * P.d + e];
      for (int sl = s0 + 1; sl < s1; ++sl) s += ws[(size_t)sl * J.bn * P.d + e];
      out[c0 * P.ld + e] = s;
    }
  }
}

template <int DIST, typename T>
cudaError_t launch_jki_t(const ApplyArgs& a, const JkiPlanView& J, cudaStream_t stream) {
  const size_t smem = jki_smem_bytes<T>(J.bn);
  cudaError_t e = cudaFuncSetAttribute(sk_jki_kernel<DIST, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // scratch (stream-ordered): values in CSR order, then the workspace slots of split blocks
  const size_t vbytes = ((size_t)J.n_ent * sizeof(T) + 255) & ~(size_t)255;
  char* scratch = nullptr;
  e = cudaMallocAsync((void**)&scratch, vbytes + (size_t)J.n_slots * J.bn * a.d * sizeof(T), stream);
  if (e != cudaSuccess) return e;
  T* vcsr = reinterpret_cast<T*>(scratch);
  T* ws = reinterpret_cast<T*>(scratch + vbytes);
  sk_jki_gather_kernel<T><<<148 * 8, 256, 0, stream>>>(reinterpret_cast<const T*>(a.vals), J.ent_p, J.n_ent, vcsr);
  e = cudaGetLastError();
  if (e == cudaSuccess) {
    sk_jki_kernel<DIST, T><<<(unsigned)J.n_items, kJThreads, smem, stream>>>(a, J, vcsr, ws);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && J.n_slots > 0) {
    sk_jki_finish_kernel<T><<<148 * 4, 256, 0, stream>>>(a, J, ws);
    e = cudaGetLastError();
  }
  const cudaError_t e2 = cudaFreeAsync(scratch, stream);
  return e == cudaSuccess ? e2 : e;
}

}  // namespace

int jki_block_cols(int dtype) {
  // the largest b_n whose accumulator + staging fits the 227 KB of shared memory per CTA
  return dtype == 0 ? 1024 : 2048;
}

size_t jki_smem(int dtype, int bn) { return dtype == 0 ? jki_smem_bytes<double>(bn) : jki_smem_bytes<float>(bn); }

cudaError_t launch_apply_jki(int dist, int dtype, const ApplyArgs& a, const JkiPlanView& J, cudaStream_t stream) {
  if (J.n_items == 0) return cudaSuccess;
  if (dist == 1) return dtype == 0 ? launch_jki_t<1, double>(a, J, stream) : launch_jki_t<1, float>(a, J, stream);
  if (dist == 2) return dtype == 0 ? launch_jki_t<2, double>(a, J, stream) : launch_jki_t<2, float>(a, J, stream);
  return cudaErrorInvalidValue;
}

}  // namespace sk
