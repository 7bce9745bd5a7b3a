// kernels.h -- internal launcher interface between the C ABI (sketch_api.cu) and the
// sm_100a kernels (sketch_kernels.cu).  Not part of the public boundary.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "philox.cuh"

namespace sk {

// Threads per CTA of the fused apply kernels: 16 warps.
constexpr int kWarps = 16;
constexpr int kThreads = kWarps * 32;
// Rows of Â owned by one warp.  Rademacher: 32 rows per lane (one 32-bit Philox word per
// lane per nonzero).  Uniform / Gaussian: 16 rows per lane (8 Philox blocks per nonzero).
constexpr int kRowsPerWarpRad = 1024;
#ifndef SK_PAIR_ROWS_PER_WARP
#define SK_PAIR_ROWS_PER_WARP 512
#endif
constexpr int kRowsPerWarpPair = SK_PAIR_ROWS_PER_WARP;
#ifndef SK_GAUSS_ROWS_PER_WARP
#define SK_GAUSS_ROWS_PER_WARP 256
#endif
constexpr int kRowsPerWarpGauss = SK_GAUSS_ROWS_PER_WARP;   // Gaussian: 8 rows per lane

// One CTA of work: column `col`, Â rows [row0, row0 + wd * rows_per_warp).
// The CTA's 16 warps are arranged as W_d = wd row-warps times W_k = 16 / wd slices of the
// column's nonzero stream (16 - W_d W_k warps idle when W_d does not divide 16).
struct Item {
  int32_t col;
  int32_t row0;
  int32_t wd;
  int32_t pad;
};

struct ApplyArgs {
  const int64_t* colptr;
  const int32_t* rowidx;
  const void* vals;
  void* out;
  const Item* items;
  int64_t n_items;
  int64_t d;
  int64_t ld;           // leading dimension of out (== d)
  int64_t row_offset;
  PhiloxKeys keys;
};

// Work item of the tensor-core ±1 kernel (sketch_f4.cu): column `col`, 128-row tiles
// [tile0, tile0 + ntiles); pad 0 = the whole column, 1 / 2 = first / second half of its K-steps (the
// last wave split along K; the halves add into zeroed rows).
struct TcItem {
  int32_t col;
  int32_t tile0;
  int32_t ntiles;
  int32_t pad;
};

// Longest column the tensor-core kernel takes: the digit sums |D| <= L stay exact in the f32
// accumulator (L < 2^24), and the value rounding <= L 2^-62 max|a| stays far below the fp64 parity
// bound (2^-45 |S||A| at L = 2^17).  Longer columns run on the SIMT kernel.
constexpr int64_t kTcMaxColumn = 131071;

// The tensor-core kernel, with the zeroing of the K-split rows before it and the IEEE fix-up of the
// columns it found non-finite after it.
// split_begin: first item of the K-split tail (n_items when there is none: no zeroing launch).
cudaError_t launch_apply_rad_f4(const ApplyArgs& a, const TcItem* items, int64_t n_items, int64_t split_begin,
                                bool persistent, cudaStream_t stream);

// ±1 sketch columns holding a NaN / Inf value get the IEEE result (sketch_kernels.cu): a scan of
// every column's values, one warp per column (dtype 0 = f64, 1 = f32).
cudaError_t launch_rad_ieee_fixup(int dtype, const ApplyArgs& a, int64_t n_cols, cudaStream_t stream);
int f4_tiles_per_cta();
// Algorithm 4 (jki) with full row reuse (sketch_jki.cu): vertical blocks of up to b_n columns, each
// stored row by row; a work item = (tile of kJRows rows of Â, block, range of the block's batches of
// up to kJBatch nonzero rows / kJBatchEnt entries).
constexpr int kJRows = 32;
constexpr int kJBatch = 128;
constexpr int kJBatchEnt = 512;
constexpr int kJOwners = 32;       // column owners (half-warps): column k of a block -> k mod 32
constexpr int kJOwnStride = 34;    // owner offsets per batch (33 used; 4-byte multiple for cp.async)
// An entry's descriptor as the kernel consumes it: byte offset of its accumulator row pair
// (column within block x 16 pairs x pair bytes, < 2^17) | byte offset of its S row (row slot within
// the batch x 16 pairs x pair bytes) << 17.  Pair bytes: 16 (f64), 8 (f32).
inline uint32_t jki_desc(uint32_t col, uint32_t slot, int dtype) {
  const uint32_t row_bytes = (kJRows / 2) * (dtype == 0 ? 16u : 8u);
  return col * row_bytes | (slot * row_bytes) << 17;
}
struct JBatch {
  int64_t ent0;        // first entry (in ent)
  int32_t row0;        // first nonzero row (in row_j)
  int16_t nrows;       // <= kJBatch
  int16_t block;       // vertical block
  int32_t nent;        // <= kJBatchEnt
  int32_t pad;
};
struct JItem {
  int32_t tile;        // rows [kJRows tile, +kJRows) of Â
  int32_t block;       // vertical block (an empty block's items write zeros)
  int32_t bt0, bt1;    // batches [bt0, bt1) of the block
  int32_t slot;        // workspace slot (the block's batches are split over several items), -1: write Â
};
struct JkiPlanView {
  const JItem* items;
  int64_t n_items;
  const JBatch* batches;
  const uint16_t* own;       // [n_batches][kJOwnStride]: entry ranges of the owners within the batch
  const int32_t* row_j;      // local row index of each nonzero row of each block
  const uint32_t* ent_p;     // value index of each entry (block CSR order)
  const uint32_t* ent_desc;  // jki_desc(column within block, row slot within batch, dtype)
  const int32_t* blk_slot;   // [n_blocks + 1]: workspace slots of block b ([s0, s1), empty if unsplit)
  int64_t n;                 // columns of the plan
  int32_t bn;                // columns per block
  int32_t n_blocks;
  int64_t n_slots;           // workspace slots (bn x d each)
  int64_t n_ent;             // entries (= nnz)
};
// Stream-ordered scratch from the library's own memory pool on the current device (its release
// threshold keeps freed memory mapped, so per-apply scratch does not re-map pages every call).
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t stream);
// cudaFuncSetAttribute(kernel, MaxDynamicSharedMemorySize, bytes) once per (kernel, device) and size:
// the call costs several µs of host time, which a small apply (c1) otherwise pays every launch.
cudaError_t set_max_dynamic_smem(const void* kernel, size_t bytes);
int jki_block_cols(int dtype);
size_t jki_smem(int dtype, int bn);
cudaError_t launch_apply_jki(int dist, int dtype, const ApplyArgs& a, const JkiPlanView& J, cudaStream_t stream);

// dist: 0 = Rademacher, 1 = uniform, 2 = Gaussian; dtype: 0 = f64, 1 = f32.
cudaError_t launch_apply(int dist, int dtype, const ApplyArgs& a, cudaStream_t stream);

cudaError_t launch_fill_s(int dist, int dtype, uint64_t seed, int64_t i0, int64_t i1, int64_t j0,
                          int64_t j1, void* out, int64_t ld, cudaStream_t stream);

// *count += number of distinct values in rowidx[p0, p1); bitmap (>= m bits) must be zero on entry
// and is left with those rows' bits set.
cudaError_t launch_distinct_rows(const int32_t* rowidx, int64_t p0, int64_t p1, uint32_t* bitmap,
                                 unsigned long long* count, cudaStream_t stream);

// Sets *flag (device int) nonzero if some rowidx is outside [0, m).
cudaError_t launch_validate_rows(const int32_t* rowidx, int64_t nnz, int64_t m, int* flag,
                                 cudaStream_t stream);

// max_p |v_p| over v[pb, pe) as the bit pattern of |v| (sign cleared), per thread tid of nt: the
// integer order of these patterns is the order of |v| with NaN > Inf > finite, so a NaN anywhere
// shows up in the maximum (fmax would drop it).  16-byte loads, 8 values in flight per thread.
__device__ __forceinline__ unsigned long long col_absmax_bits(const double* __restrict__ v, int64_t pb, int64_t pe,
                                                              int tid, int nt) {
  constexpr unsigned long long kAbs = 0x7FFFFFFFFFFFFFFFull;
  auto ab = [](double x) { return (unsigned long long)__double_as_longlong(x) & kAbs; };
  unsigned long long m0 = 0, m1 = 0, m2 = 0, m3 = 0;
  if ((reinterpret_cast<uintptr_t>(v) & 15) != 0) {
    for (int64_t p = pb + tid; p < pe; p += nt) m0 = max(m0, ab(__ldg(v + p)));
    return m0;
  }
  int64_t a = (pb + 1) & ~(int64_t)1;            // first 16-byte aligned index >= pb
  if (a > pe) a = pe;
  const int64_t n2 = (pe - a) >> 1;              // double2 body [a, a + 2 n2)
  if (tid == 0 && pb < a) m0 = ab(__ldg(v + pb));
  if (tid == nt - 1 && a + 2 * n2 < pe) m1 = ab(__ldg(v + a + 2 * n2));
  const double2* v2 = reinterpret_cast<const double2*>(v + a);
  int64_t i = tid;
  for (; i + 3 * (int64_t)nt < n2; i += 4 * (int64_t)nt) {
    const double2 x0 = __ldg(v2 + i), x1 = __ldg(v2 + i + nt), x2 = __ldg(v2 + i + 2 * nt), x3 = __ldg(v2 + i + 3 * nt);
    m0 = max(m0, max(ab(x0.x), ab(x0.y)));
    m1 = max(m1, max(ab(x1.x), ab(x1.y)));
    m2 = max(m2, max(ab(x2.x), ab(x2.y)));
    m3 = max(m3, max(ab(x3.x), ab(x3.y)));
  }
  for (; i < n2; i += nt) {
    const double2 x0 = __ldg(v2 + i);
    m0 = max(m0, max(ab(x0.x), ab(x0.y)));
  }
  return max(max(m0, m1), max(m2, m3));
}

// IEEE result of column k of a ±1 sketch when its values hold a NaN or an Inf (one warp): every
// entry of Â[:, k] is then non-finite, and IEEE addition in ANY order gives NaN if a term is NaN or
// both +Inf and -Inf terms occur, else the sign of the infinite terms -- the oracle's sequential
// sum.  Lane = row within a 32-row chunk; one Philox block per (non-finite value, chunk).  Returns
// without writing when the column is finite.  Rare path.
template <typename T>
__device__ __forceinline__ void rad_ieee_fix_column(const ApplyArgs& P, int64_t k) {
  constexpr unsigned kAll = 0xFFFFFFFFu;
  const int lane = threadIdx.x & 31;
  const T* vals = reinterpret_cast<const T*>(P.vals);
  const int64_t pb = P.colptr[k], pe = P.colptr[k + 1];
  bool bad = false;
  for (int64_t p = pb + lane; p < pe; p += 32) bad |= !isfinite(vals[p]);
  if (!__any_sync(kAll, bad)) return;
  T* outc = reinterpret_cast<T*>(P.out) + k * P.ld;
  for (int64_t r0 = 0; r0 < P.d; r0 += 32) {
    const int64_t row = r0 + lane;
    uint32_t f = 0;                                    // 1: a +Inf term, 2: a -Inf term, 4: a NaN
    for (int64_t p0 = pb; p0 < pe; p0 += 32) {
      const T v = p0 + lane < pe ? vals[p0 + lane] : T(0);
      const int32_t j = p0 + lane < pe ? P.rowidx[p0 + lane] : 0;
      if (__any_sync(kAll, isnan(v))) f |= 4u;
      for (unsigned m = __ballot_sync(kAll, isinf(v)); m; m &= m - 1) {
        const int s = __ffs(m) - 1;
        const T vi = __shfl_sync(kAll, v, s);
        const uint32_t jr = (uint32_t)__shfl_sync(kAll, j, s);
        const uint4 x = s_block((uint32_t)(row >> 7), (uint64_t)P.row_offset + jr, P.keys);
        const int t = (int)((row >> 5) & 3);
        const uint32_t w = t == 0 ? x.x : t == 1 ? x.y : t == 2 ? x.z : x.w;
        const uint32_t neg = ((w >> (row & 31)) & 1u) ^ (vi < T(0) ? 1u : 0u);   // S = -1 where the bit is set
        f |= neg ? 2u : 1u;
      }
    }
    if (row < P.d) outc[row] = (f & 4u) || f == 3u ? T(NAN) : (f == 1u ? T(INFINITY) : T(-INFINITY));
  }
}

}  // namespace sk
