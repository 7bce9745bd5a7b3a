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
//  * work item = (tile of kJRows = 32 rows of Â, block, range of the block's row batches): the CTA
//    keeps the 32 x b_n accumulator of its tile in shared memory (fp64: 256 B per column, b_n = 384);
//  * a batch = up to kJBatch = 128 nonzero rows (<= kJBatchEnt = 512 entries).  Stage (all 512
//    threads): S[tile rows, j] for the batch's rows -- 2048 Philox blocks, four per thread -- into
//    shared memory, and the batch's entries (column, row slot, value);
//  * scatter: half-warp h (32 per CTA) owns the block's columns k = h mod 32 and applies the batch's
//    entries of its columns in row order, lane i updating rows 2i, 2i+1 (the two entries of one
//    Philox block; one 16-byte shared load of S, one load and one store of the accumulator pair per
//    entry): acc[k][2i..2i+1] += S[slot][2i..2i+1] a.  Entries of one column are applied by one
//    half-warp in a fixed order, so results are deterministic;
//  * latency: a first kernel gathers the values into the blocks' CSR order (vals_csr[e] = vals[p_e],
//    coalesced writes), so a batch's inputs are contiguous ranges, copied by cp.async into a ring
//    of shared-memory slots kJDepth = 3 batches ahead; S is double-buffered, so the scatter of batch
//    b and the stage of batch b+1 run between the same two barriers (one __syncthreads per batch) and
//    one warp's scatter latency hides under the other warps' Philox work;
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

static_assert(kJRows == 32, "a half-warp lane owns the two rows of one Philox block");
constexpr int kJQ = kJRows / 2;      // Philox blocks per (tile, row j) = lanes of a half-warp

template <typename T> struct Vec2;
template <> struct Vec2<double> { using type = double2; };
template <> struct Vec2<float> { using type = float2; };

// entry descriptor (jki_desc, kernels.h): accumulator byte offset (< b_n x 256 <= 2^17) | S byte offset << 17
static_assert(kJBatch * kJQ * 16 <= (1 << 15), "S offset must fit 15 bits");

// The inputs of a batch (its nonzero rows, entries and owner ranges) arrive by cp.async into a ring of
// kJRing slots, kJDepth batches ahead of the batch being staged (the loads are independent of the
// compute, so their latency hides under kJDepth batches of Philox / scatter work); the batch headers
// arrive 2 kJDepth ahead, so every address a copy needs is already in shared memory.
constexpr int kJDepth = 3;
constexpr int kJRing = kJDepth + 1;
constexpr int kJHdrRing = 8;
static_assert(kJHdrRing >= 2 * kJDepth && kJDepth >= 2, "ring sizes");

template <typename T>
struct JSlot {                                   // byte layout of one ring slot
  // entry records [kJBatchEnt]: descriptor at +0, value at +sizeof(T) (one 16-byte load in fp64)
  static constexpr int ent = 2 * (int)sizeof(T);
  static constexpr int ents = 0;
  static constexpr int rj = ents + kJBatchEnt * ent;               // int32 [kJBatch]
  static constexpr int own = rj + kJBatch * 4;                     // uint16 [kJOwnStride]
  static constexpr int bytes = (own + kJOwnStride * 2 + 15) & ~15;
};

template <typename T>
constexpr size_t jki_smem_bytes(int bn) {
  return (size_t)bn * kJRows * sizeof(T)                 // accumulator
         + 2 * (size_t)kJBatch * kJRows * sizeof(T)     // S of two batches
         + (size_t)kJRing * JSlot<T>::bytes             // input ring
         + kJHdrRing * sizeof(JBatch)                   // batch headers
         + kJLogBytes;
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

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

constexpr int kJSlotsPerThread = kJBatch * kJQ / kJThreads;   // 4 Philox blocks per thread per batch
static_assert(kJBatchEnt <= kJThreads && kJBatch <= kJThreads && sizeof(JBatch) == 24, "one copy per thread");

template <int DIST, typename T>
__global__ void __launch_bounds__(kJThreads, 1) sk_jki_kernel(const ApplyArgs P, const JkiPlanView J,
                                                               const T* __restrict__ vcsr, T* __restrict__ ws) {
  extern __shared__ __align__(16) unsigned char smem[];
  using V2 = typename Vec2<T>::type;
  const JItem it = J.items[blockIdx.x];
  const int64_t c0 = (int64_t)it.block * J.bn;
  const int nbc = (int)min((int64_t)J.bn, J.n - c0);              // columns of this block
  V2* acc = reinterpret_cast<V2*>(smem);                           // [nbc][kJQ] row pairs
  V2* S = acc + (size_t)J.bn * kJQ;                                // [2][kJBatch][kJQ]
  unsigned char* ring = reinterpret_cast<unsigned char*>(S + 2 * kJBatch * kJQ);   // [kJRing] slots
  JBatch* hdr = reinterpret_cast<JBatch*>(ring + kJRing * JSlot<T>::bytes);        // [kJHdrRing]
  double* logtab = reinterpret_cast<double*>(hdr + kJHdrRing);
  const double* mylog = logtab + (threadIdx.x & (kJLogRep - 1));
  const int tid = threadIdx.x;
  const uint32_t q0 = (uint32_t)it.tile * kJQ;                     // Philox block of the tile's first row
  const int ql = tid & (kJQ - 1);
  const int bt0 = it.bt0, bt1 = it.bt1;

  for (int e = tid; e < nbc * kJQ; e += kJThreads) acc[e] = V2{T(0), T(0)};
  if constexpr (DIST == 2) jki_fill_logtab(logtab);

  auto slot_of = [&](int x) { return ring + ((x - bt0) % kJRing) * JSlot<T>::bytes; };
  auto issue_hdr = [&](int x) {                                    // header of batch x (3 x 8 bytes)
    if (tid < 3 && x < bt1)
      cp_async8(reinterpret_cast<char*>(hdr + (x - bt0) % kJHdrRing) + 8 * tid,
                reinterpret_cast<const char*>(J.batches + x) + 8 * tid);
  };
  auto issue_data = [&](int x) {                                   // inputs of batch x (header visible)
    if (x >= bt1) return;
    const JBatch& B = hdr[(x - bt0) % kJHdrRing];
    unsigned char* sl = slot_of(x);
    if (tid < B.nent) {
      unsigned char* rec = sl + JSlot<T>::ents + JSlot<T>::ent * tid;
      cp_async4(rec, J.ent_desc + B.ent0 + tid);
      if constexpr (sizeof(T) == 8) cp_async8(rec + 8, vcsr + B.ent0 + tid);
      else cp_async4(rec + 4, vcsr + B.ent0 + tid);
    }
    if (tid < B.nrows) cp_async4(sl + JSlot<T>::rj + 4 * tid, J.row_j + B.row0 + tid);
    if (tid < kJOwnStride / 2) cp_async4(sl + JSlot<T>::own + 4 * tid, J.own + (int64_t)x * kJOwnStride + 2 * tid);
  };
  // stage: S[tile rows, j] of batch x's rows -> S buffer b (2 Philox blocks per thread)
  auto stage = [&](int x, int b) {
    const int nrows = hdr[(x - bt0) % kJHdrRing].nrows;
    const int32_t* rj = reinterpret_cast<const int32_t*>(slot_of(x) + JSlot<T>::rj);
    V2* Sb = S + b * (kJBatch * kJQ);
    if (nrows == kJBatch) {
      // a full batch: the kJSlotsPerThread blocks as independent chains the scheduler interleaves
      uint4 x4[kJSlotsPerThread];
#pragma unroll
      for (int h = 0; h < kJSlotsPerThread; ++h)
        x4[h] = s_block(q0 + ql, (uint64_t)P.row_offset + (uint32_t)rj[(tid >> 4) + (kJThreads / kJQ) * h], P.keys);
#pragma unroll
      for (int h = 0; h < kJSlotsPerThread; ++h) {
        T v0, v1;
        jki_entries<DIST, T>(x4[h], mylog, v0, v1);
        Sb[((tid >> 4) + (kJThreads / kJQ) * h) * kJQ + ql] = V2{v0, v1};
      }
    } else {
      // a partial batch (rows with many entries): only the threads of its rows generate
#pragma unroll
      for (int h = 0; h < kJSlotsPerThread; ++h) {
        const int slot = (tid >> 4) + (kJThreads / kJQ) * h;
        if (slot < nrows) {
          const uint4 x4 = s_block(q0 + ql, (uint64_t)P.row_offset + (uint32_t)rj[slot], P.keys);
          T v0, v1;
          jki_entries<DIST, T>(x4, mylog, v0, v1);
          Sb[slot * kJQ + ql] = V2{v0, v1};
        }
      }
    }
  };

  if (bt0 < bt1) {
    for (int k = 0; k < 2 * kJDepth; ++k) issue_hdr(bt0 + k);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    for (int k = 0; k < kJDepth; ++k) issue_data(bt0 + k);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();                                               // (also the log table)
    stage(bt0, 0);
  }
  __syncthreads();
  const int hw = tid >> 4, i = tid & 15;                           // half-warp = column owner, lane = row pair
  for (int x = bt0; x < bt1; ++x) {
    const int b = (x - bt0) & 1;
    issue_hdr(x + 2 * kJDepth);
    issue_data(x + kJDepth);
    cp_async_commit();
    {                                                              // scatter batch x
      const unsigned char* sl = slot_of(x);
      const unsigned char* er = sl + JSlot<T>::ents;
      const uint16_t* own = reinterpret_cast<const uint16_t*>(sl + JSlot<T>::own);
      const char* Sb = reinterpret_cast<const char*>(S + b * (kJBatch * kJQ) + i);
      char* acci = reinterpret_cast<char*>(acc + i);
      const int e1 = own[hw + 1];
      // an owner's entries come in row order, so consecutive entries of one row reuse the S pair
      // already in registers (one record load + the accumulator load and store per entry)
      uint32_t prev = 0xFFFFFFFFu;
      V2 sv{T(0), T(0)};
      for (int e = own[hw]; e < e1; ++e) {
        uint32_t dsc;
        T a;
        if constexpr (sizeof(T) == 8) {
          const uint4 r = *reinterpret_cast<const uint4*>(er + 16 * e);
          dsc = r.x;
          a = __hiloint2double((int)r.w, (int)r.z);
        } else {
          const uint2 r = *reinterpret_cast<const uint2*>(er + 8 * e);
          dsc = r.x;
          a = __uint_as_float(r.y);
        }
        V2* slot = reinterpret_cast<V2*>(acci + (dsc & 0x1FFFFu));
        const uint32_t soff = dsc >> 17;
        if (soff != prev) {
          sv = *reinterpret_cast<const V2*>(Sb + soff);
          prev = soff;
        }
        V2 av = *slot;
        av.x = fma(sv.x, a, av.x);
        av.y = fma(sv.y, a, av.y);
        *slot = av;
      }
    }
    if (x + 1 < bt1) stage(x + 1, b ^ 1);
    cp_async_wait<kJDepth - 2>();                                  // batch x + 2's inputs, header x + D + 1
    __syncthreads();
  }
  cp_async_wait<0>();

  // the tile's rows [32 tile, +32) of the block's columns: to Â, or to this item's workspace slot
  const int64_t row0 = (int64_t)it.tile * kJRows;
  T* dst = it.slot < 0 ? reinterpret_cast<T*>(P.out) + c0 * P.ld
                       : ws + (size_t)it.slot * (size_t)J.bn * (size_t)P.d;
  const T* accs = reinterpret_cast<const T*>(acc);
  for (int e = tid; e < nbc * kJRows; e += kJThreads) {
    const int c = e / kJRows, r = e % kJRows;
    if (row0 + r < P.d) dst[(int64_t)c * P.d + row0 + r] = accs[e];
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
  cudaError_t e = set_max_dynamic_smem((const void*)sk_jki_kernel<DIST, T>, smem);
  if (e != cudaSuccess) return e;
  // scratch (stream-ordered, library pool): values in CSR order, then the workspace slots of split blocks
  const size_t vbytes = ((size_t)J.n_ent * sizeof(T) + 255) & ~(size_t)255;
  char* scratch = nullptr;
  e = scratch_alloc((void**)&scratch, vbytes + (size_t)J.n_slots * J.bn * a.d * sizeof(T), stream);
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
  // (and whose accumulator byte offsets fit the 17 bits of the descriptor): 96 KB of accumulator next to
  // the 64 KB (f64) double-buffered S of 128-row batches
  return dtype == 0 ? 384 : 768;
}

size_t jki_smem(int dtype, int bn) { return dtype == 0 ? jki_smem_bytes<double>(bn) : jki_smem_bytes<float>(bn); }

cudaError_t launch_apply_jki(int dist, int dtype, const ApplyArgs& a, const JkiPlanView& J, cudaStream_t stream) {
  if (J.n_items == 0) return cudaSuccess;
  if (dist == 1) return dtype == 0 ? launch_jki_t<1, double>(a, J, stream) : launch_jki_t<1, float>(a, J, stream);
  if (dist == 2) return dtype == 0 ? launch_jki_t<2, double>(a, J, stream) : launch_jki_t<2, float>(a, J, stream);
  return cudaErrorInvalidValue;
}

}  // namespace sk
