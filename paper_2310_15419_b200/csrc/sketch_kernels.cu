// sketch_kernels.cu -- fused on-the-fly-RNG sparse sketch kernels for sm_100a.
//
// Computes Â[:, k] = Σ_{p in column k} S[:, j_p] · a_p with S regenerated
// from Philox for every stored nonzero: the loop order of Algorithm 3 ("kji"),
// mapped to the GPU as follows (DESIGN.md §"Kernels"):
//   * the outer blocking of Algorithm 1 becomes the grid: one CTA per work
//     item = (column k, tile of Â rows), items ordered longest-first by the plan;
//   * the d-dimension of a tile is split over W_d warps, and the column's nonzero stream over
//     W_k = 16 / W_d warps (each warp a contiguous slice);
//   * accumulators live in registers: a lane owns 32 consecutive Â rows for ±1 (exactly one
//     32-bit Philox word per nonzero) or 16 rows for uniform / Gaussian (8 Philox blocks);
//   * the W_k partial tiles are reduced in shared memory in a fixed order and the Â tile is
//     written to HBM exactly once, coalesced (Algorithm 1's Â = 0 then accumulate,
//     PAPER.md:83, becomes "overwrite with the full sum").
// No tensor cores: per column this is a matrix-vector product with a freshly generated
// matrix, not a dense contraction.
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "kernels.h"
#include "philox.cuh"

namespace sk {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kXchWords = 5;                                   // padded 4-word exchange slot
constexpr int kXchBytes = kWarps * 32 * kXchWords * 4;         // 10 KiB
constexpr int kRadPad = 33;                                    // 32 rows per lane + 1 pad

template <typename T>
__device__ __forceinline__ T ldg_val(const void* vals, int64_t p) {
  return __ldg(reinterpret_cast<const T*>(vals) + p);
}

// Sign application for the 32 rows a lane owns, one 32-bit Philox word w per nonzero a.
//  fp64:  acc[b] += (bit b of w) ? -a : a.  Only the high word of ±a differs, so each
//         element is one SEL (predicate from R2P, 8 bits per R2P) + one DADD; the select is
//         written in PTX because ptxas otherwise emits a 2-instruction shift/xor or a
//         2-word FSEL per element.
//  fp32:  the "T - 2P" form Â = Σ a - 2 Σ_{bit=1} a: one predicated FADD per element
//         (acc holds P; the lane-uniform column total T is kept separately).
__device__ __forceinline__ void apply_signs(double (&acc)[32], uint32_t w, double a) {
  // high word of ±a selected per element (SEL, predicate from R2P), shared low word, DADD
  const int lo = __double2loint(a), hi = __double2hiint(a), nhi = hi ^ (int)0x80000000;
#pragma unroll
  for (int b = 0; b < 32; ++b) {
    int h;
    asm("{.reg .pred p; .reg .b32 t; and.b32 t, %1, %4; setp.ne.u32 p, t, 0; selp.b32 %0, %2, %3, p;}"
        : "=r"(h) : "r"(w), "r"(nhi), "r"(hi), "r"(1u << b));
    acc[b] += __hiloint2double(h, lo);
  }
}

__device__ __forceinline__ void apply_signs(float (&acc)[32], uint32_t w, float a) {
#pragma unroll
  for (int b = 0; b < 32; ++b)
    if ((w >> b) & 1u) acc[b] += a;
}

template <typename T>
__device__ __forceinline__ T finish_sign_sum(T acc, T total) {
  if constexpr (sizeof(T) == 8) { return acc; }
  else { return fmaf(-2.0f, acc, total); }       // T - 2P
}

// ------------------------------------------------------------------ ±1 (Rademacher)
//
// Lane l of a warp owns Â rows warp_row0 + 32 l + b (b = 0..31), i.e. word t = l % 4 of
// Philox block q = warp_row0/128 + l/4.  The four lanes of a quad need the same block q for
// every nonzero, so they split the RNG work: for a group of 4 nonzeros, lane t of the quad
// generates block q of nonzero 4u + t, and a 4x4 word transpose through shared memory hands
// every lane its own word of all four blocks.  One Philox call per 128 (row, nonzero) pairs.
// fp32 needs 32 accumulator registers, so two CTAs fit per SM (one CTA's prologue / reduction /
// store overlaps the other's main loop); fp64 needs 64 and runs one CTA per SM.
template <typename T>
__global__ void __launch_bounds__(kThreads, sizeof(T) == 4 ? 2 : 1) sk_rad_kernel(const ApplyArgs P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Item it = P.items[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int WD = it.wd, WK = kWarps / WD;              // warps >= WD*WK get an empty slice
  const int wd = warp % WD, wk = warp / WD;
  const int64_t pb = P.colptr[it.col], pe = P.colptr[it.col + 1];
  const int64_t L = pe - pb;
  const int64_t s0 = wk < WK ? pb + (L * wk) / WK : pe, s1 = wk < WK ? pb + (L * (wk + 1)) / WK : pe;
  const int64_t warp_row0 = (int64_t)it.row0 + (int64_t)wd * kRowsPerWarpRad;
  const uint32_t q = (uint32_t)(warp_row0 >> 7) + (uint32_t)(lane >> 2);
  const int t = lane & 3, g = lane >> 2;
  uint32_t* xch = reinterpret_cast<uint32_t*>(smem) + warp * (32 * kXchWords);

  T acc[32];
#pragma unroll
  for (int b = 0; b < 32; ++b) acc[b] = T(0);
  T total = T(0);   // fp32 "T - 2P" form only
  for (int64_t p = s0; p < s1; p += 32) {
    const int cnt = (int)((s1 - p) < 32 ? (s1 - p) : 32);
    int32_t jl = 0;
    T al = T(0);
    if (lane < cnt) {
      jl = __ldg(P.rowidx + p + lane);
      al = ldg_val<T>(P.vals, p + lane);
    }
    const int ngroups = (cnt + 3) >> 2;
    for (int u = 0; u < ngroups; ++u) {
      const uint32_t jr = (uint32_t)__shfl_sync(kFull, jl, 4 * u + t);
      const uint64_t J = (uint64_t)P.row_offset + jr;
      const uint4 x = s_block(q, J, P.keys);
      xch[lane * kXchWords + 0] = x.x;
      xch[lane * kXchWords + 1] = x.y;
      xch[lane * kXchWords + 2] = x.z;
      xch[lane * kXchWords + 3] = x.w;
      __syncwarp();
      uint32_t w[4];
#pragma unroll
      for (int s = 0; s < 4; ++s) w[s] = xch[(4 * g + s) * kXchWords + t];
      __syncwarp();
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const T a = __shfl_sync(kFull, al, 4 * u + s);   // 0 past cnt: adds ±0
        total += a;
        apply_signs(acc, w[s], a);
      }
    }
  }

  // Fixed-order reduction of the W_k partial tiles, then one coalesced store per row.
  T* red = reinterpret_cast<T*>(smem + kXchBytes);
  T* mine = red + warp * (32 * kRadPad) + lane * kRadPad;
#pragma unroll
  for (int b = 0; b < 32; ++b) mine[b] = finish_sign_sum(acc[b], total);
  __syncthreads();
  T* outc = reinterpret_cast<T*>(P.out) + (int64_t)it.col * P.ld;
  const int rows = WD * kRowsPerWarpRad;
  for (int r = threadIdx.x; r < rows; r += kThreads) {
    const int64_t row = (int64_t)it.row0 + r;
    if (row >= P.d) break;
    const int rwd = r >> 10, rr = r & 1023;
    const int off = (rr >> 5) * kRadPad + (rr & 31);
    T s = red[rwd * (32 * kRadPad) + off];
    for (int kk = 1; kk < WK; ++kk) s += red[(kk * WD + rwd) * (32 * kRadPad) + off];
    outc[row] = s;
  }
}

// ------------------------------------------------------------------ uniform / Gaussian / uniform24
//
// Lane l owns Â rows warp_row0 + 16 l + e (e = 0..15) = entries of the 16/E Philox blocks
// q = (warp_row0 + 16 l)/E + h; each block yields E entries (E = 2 for uniform / Gaussian, 4 for
// uniform24), so a lane generates exactly the S entries it consumes (no exchange).
template <int DIST> constexpr int pair_E() { return DIST == 3 ? 4 : 2; }
// logtab / STRIDE: the -2 log table (philox.cuh bm_m2log_u53); sctab / SCREP: the sin / cos table
// (bm_sincos); Gaussian only.
template <int DIST, typename T, int STRIDE = 0, int SCREP = kScRep>
__device__ __forceinline__ void pair_entries(const uint4 x, T& v0, T& v1, const double* __restrict__ logtab,
                                             const double* __restrict__ sctab = nullptr) {
  if constexpr (DIST == 1) {
    const double d0 = uniform53(x.x, x.y), d1 = uniform53(x.z, x.w);
    if constexpr (sizeof(T) == 8) { v0 = d0; v1 = d1; }
    else { v0 = __double2float_rn(d0); v1 = __double2float_rn(d1); }
  } else {
    double g0, g1;
    gaussian_pair_fast<STRIDE, SCREP>(x, logtab, sctab, g0, g1);
    if constexpr (sizeof(T) == 8) { v0 = g0; v1 = g1; }
    else { v0 = __double2float_rn(g0); v1 = __double2float_rn(g1); }
  }
}

template <int DIST, typename T, int STRIDE = 0, int SCREP = kScRep>
__device__ __forceinline__ void block_entries(const uint4 x, T (&v)[pair_E<DIST>()], const double* __restrict__ logtab,
                                              const double* __restrict__ sctab = nullptr) {
  if constexpr (DIST == 3) {
    v[0] = (T)uniform24(x.x); v[1] = (T)uniform24(x.y); v[2] = (T)uniform24(x.z); v[3] = (T)uniform24(x.w);
  } else {
    pair_entries<DIST, T, STRIDE, SCREP>(x, v[0], v[1], logtab, sctab);
  }
}

// Rows per lane: 16 (uniform, uniform24: kRowsPerWarpPair = 512 per warp) or 8 (Gaussian:
// kRowsPerWarpGauss = 256; fewer live accumulators leave the Box-Muller chains registers:
// c3 16.1 -> 15.0 ms, while uniform prefers 16: 2.71 vs 2.82 ms on c2).
// Gaussian tables in shared memory: the -2 log table as one copy in 32-byte rows (a 16 + 8 byte load
// per pair; the rows' bank groups conflict, but the conflict-free replicated layout -- 3 loads of
// 8 bytes from a 49.5 KB table -- measured slower, c3 13.53 vs 13.05 ms), and the sin / cos table
// replicated kScRep = 8 times (conflict-free 16-byte loads, instead of ~8-wavefront L1 gathers of
// kBmSinCosTab: 13.05 vs 13.27 ms).  One CTA per item (a persistent grid-stride variant with the
// tables filled once per SM measured 15.2 ms: its static item assignment leaves the SMs unbalanced).
constexpr int kGaussScRep = kScRep;
template <int DIST> constexpr int pair_rows() { return (DIST == 2 ? kRowsPerWarpGauss : kRowsPerWarpPair) / 32; }

// One work item of the uniform / Gaussian / uniform24 kernel (the CTA's 16 warps; `red` = the
// reduction area).  Lane l owns Â rows row0 + 32 kPairRows w_d + kPairRows l + e.
template <int DIST, typename T>
__device__ __forceinline__ void pair_item(const ApplyArgs& P, const Item it, T* red, const double* __restrict__ logtab,
                                          const double* __restrict__ sctab) {
  constexpr int kPairRows = pair_rows<DIST>(), kPairPad = kPairRows + 1, kRowsPerWarp = 32 * kPairRows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int WD = it.wd, WK = kWarps / WD;              // warps >= WD*WK get an empty slice
  const int wd = warp % WD, wk = warp / WD;
  const int64_t pb = P.colptr[it.col], pe = P.colptr[it.col + 1];
  const int64_t L = pe - pb;
  const int64_t s0 = wk < WK ? pb + (L * wk) / WK : pe, s1 = wk < WK ? pb + (L * (wk + 1)) / WK : pe;
  const int64_t lane_row0 = (int64_t)it.row0 + (int64_t)wd * kRowsPerWarp + kPairRows * lane;
  constexpr int kE = pair_E<DIST>();
  const uint32_t q0 = (uint32_t)(lane_row0 / kE);
  // Lanes whose rows all lie past d skip generation (their results are never stored).
  const bool active = lane_row0 < P.d;

  T acc[kPairRows];
#pragma unroll
  for (int e = 0; e < kPairRows; ++e) acc[e] = T(0);

  for (int64_t p = s0; p < s1; p += 32) {
    const int cnt = (int)((s1 - p) < 32 ? (s1 - p) : 32);
    int32_t jl = 0;
    T al = T(0);
    if (lane < cnt) {
      jl = __ldg(P.rowidx + p + lane);
      al = ldg_val<T>(P.vals, p + lane);
    }
    for (int s = 0; s < cnt; ++s) {
      const uint32_t jr = (uint32_t)__shfl_sync(kFull, jl, s);
      const T a = __shfl_sync(kFull, al, s);
      if (!active) continue;
      const uint64_t J = (uint64_t)P.row_offset + jr;
      if constexpr (DIST == 2) {
        // (two scalars per block: this form schedules better than the array form, 16.1 vs 16.8 ms on c3)
#pragma unroll
        for (int h = 0; h < kPairRows / 2; ++h) {
          const uint4 x = s_block(q0 + h, J, P.keys);
          T v0, v1;
          pair_entries<DIST, T, 0, kGaussScRep>(x, v0, v1, logtab, sctab);
          acc[2 * h] = fma(v0, a, acc[2 * h]);
          acc[2 * h + 1] = fma(v1, a, acc[2 * h + 1]);
        }
      } else {
#pragma unroll
      for (int h = 0; h < kPairRows / kE; ++h) {
        const uint4 x = s_block(q0 + h, J, P.keys);
        T v[kE];
        block_entries<DIST, T>(x, v, logtab);
#pragma unroll
        for (int t = 0; t < kE; ++t) acc[kE * h + t] = fma(v[t], a, acc[kE * h + t]);
      }
      }
    }
  }

  T* mine = red + warp * (32 * kPairPad) + lane * kPairPad;
#pragma unroll
  for (int e = 0; e < kPairRows; ++e) mine[e] = acc[e];
  __syncthreads();
  T* outc = reinterpret_cast<T*>(P.out) + (int64_t)it.col * P.ld;
  const int rows = WD * kRowsPerWarp;
  for (int r = threadIdx.x; r < rows; r += kThreads) {
    const int64_t row = (int64_t)it.row0 + r;
    if (row >= P.d) break;
    const int rwd = r / kRowsPerWarp, rr = r % kRowsPerWarp;
    const int off = (rr / kPairRows) * kPairPad + (rr % kPairRows);
    T s = red[rwd * (32 * kPairPad) + off];
    for (int kk = 1; kk < WK; ++kk) s += red[(kk * WD + rwd) * (32 * kPairPad) + off];
    outc[row] = s;
  }
}

// Shared memory: reduction area, then (Gaussian) the -2 log table and the replicated sin / cos table.
template <int DIST> constexpr int pair_red_bytes() { return kWarps * 32 * (pair_rows<DIST>() + 1) * 8; }
template <int DIST> constexpr size_t pair_smem_bytes() {
  return (size_t)pair_red_bytes<DIST>() + (DIST == 2 ? (size_t)kLogTab4Bytes + kScTabRepBytes : 0);
}

// One CTA per work item (longest first).
template <int DIST, typename T>
__global__ void __launch_bounds__(kThreads, 1) sk_pair_kernel(const ApplyArgs P) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* red = reinterpret_cast<T*>(smem);
  const double* logtab = nullptr;
  const double* sctab = nullptr;
  if constexpr (DIST == 2) {
    double* lt = reinterpret_cast<double*>(smem + pair_red_bytes<DIST>());
    double* st = reinterpret_cast<double*>(smem + pair_red_bytes<DIST>() + kLogTab4Bytes);
    bm_fill_logtab4(lt);
    bm_fill_sctab(st);
    __syncthreads();
    logtab = lt;
    sctab = st + 2 * (threadIdx.x & (kScRep - 1));       // this lane's copy
  }
  pair_item<DIST, T>(P, P.items[blockIdx.x], red, logtab, sctab);
}

// ------------------------------------------------------------------ IEEE fix-up of non-finite columns
// (rad_ieee_fix_column, kernels.h): the fp32 "T - 2P" sums turn Inf - 2 Inf into NaN, so the columns
// holding a NaN / Inf are rewritten after the kernel; one warp per column.
template <typename T>
__global__ void sk_rad_ieee_fixup_kernel(const ApplyArgs P, int64_t n_cols) {
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = warp0; k < n_cols; k += nwarps) rad_ieee_fix_column<T>(P, k);
}

// ------------------------------------------------------------------ S materialisation
// One thread per Philox block (q, j); writes the block's entries that fall in [i0, i1).
template <int DIST, typename T>
__global__ void sk_fill_s_kernel(PhiloxKeys K, int64_t i0, int64_t i1, int64_t j0, int64_t j1,
                                 int64_t q0, int64_t nq, T* out, int64_t ld) {
  const int64_t total = nq * (j1 - j0);
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = q0 + idx % nq;
    const int64_t j = j0 + idx / nq;
    const uint4 x = s_block((uint32_t)q, (uint64_t)j, K);
    T* col = out + (j - j0) * ld;
    if constexpr (DIST == 0) {
      const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll 4
      for (int e = 0; e < 128; ++e) {
        const int64_t i = q * 128 + e;
        if (i >= i0 && i < i1) col[i - i0] = ((w[e >> 5] >> (e & 31)) & 1u) ? T(-1) : T(1);
      }
    } else {
      constexpr int kE = pair_E<DIST>();
      T v[kE];
      block_entries<DIST, T, 1, 0>(x, v, &kBmLogTab[0][0]);
#pragma unroll
      for (int t = 0; t < kE; ++t) {
        const int64_t i = q * kE + t;
        if (i >= i0 && i < i1) col[i - i0] = v[t];
      }
    }
  }
}

__global__ void sk_validate_rows_kernel(const int32_t* __restrict__ rowidx, int64_t nnz, int64_t m,
                                        int* flag) {
  int bad = 0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = __ldg(rowidx + p);
    bad |= (r < 0 || (int64_t)r >= m);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

template <typename K>
cudaError_t launch_items(K kernel, size_t smem, const ApplyArgs& a, cudaStream_t stream) {
  if (a.n_items == 0) return cudaSuccess;
  cudaError_t e = set_max_dynamic_smem((const void*)kernel, smem);
  if (e != cudaSuccess) return e;
  kernel<<<(unsigned)a.n_items, kThreads, smem, stream>>>(a);
  return cudaGetLastError();
}

int sm_count() {
  static const int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

}  // namespace

cudaError_t launch_apply(int dist, int dtype, const ApplyArgs& a, cudaStream_t stream) {
  const size_t rad64 = kXchBytes + (size_t)kWarps * 32 * kRadPad * 8;
  const size_t rad32 = kXchBytes + (size_t)kWarps * 32 * kRadPad * 4;
  if (dist == 0) {
    if (dtype == 1) return launch_items(sk_rad_kernel<float>, rad32, a, stream);   // + launch_rad_ieee_fixup
    return launch_items(sk_rad_kernel<double>, rad64, a, stream);
  }
  if (dist == 1) return dtype == 0 ? launch_items(sk_pair_kernel<1, double>, pair_smem_bytes<1>(), a, stream)
                                   : launch_items(sk_pair_kernel<1, float>, pair_smem_bytes<1>(), a, stream);
  if (dist == 3) return dtype == 0 ? launch_items(sk_pair_kernel<3, double>, pair_smem_bytes<3>(), a, stream)
                                   : launch_items(sk_pair_kernel<3, float>, pair_smem_bytes<3>(), a, stream);
  return dtype == 0 ? launch_items(sk_pair_kernel<2, double>, pair_smem_bytes<2>(), a, stream)
                    : launch_items(sk_pair_kernel<2, float>, pair_smem_bytes<2>(), a, stream);
}

cudaError_t launch_rad_ieee_fixup(int dtype, const ApplyArgs& a, int64_t n_cols, cudaStream_t stream) {
  const unsigned grid = (unsigned)sm_count() * 2;
  if (dtype == 0) sk_rad_ieee_fixup_kernel<double><<<grid, 256, 0, stream>>>(a, n_cols);
  else sk_rad_ieee_fixup_kernel<float><<<grid, 256, 0, stream>>>(a, n_cols);
  return cudaGetLastError();
}

cudaError_t launch_fill_s(int dist, int dtype, uint64_t seed, int64_t i0, int64_t i1, int64_t j0,
                          int64_t j1, void* out, int64_t ld, cudaStream_t stream) {
  if (i1 <= i0 || j1 <= j0) return cudaSuccess;
  const int64_t E = dist == 0 ? 128 : (dist == 3 ? 4 : 2);
  const int64_t q0 = i0 / E, q1 = (i1 + E - 1) / E, nq = q1 - q0;
  const int64_t total = nq * (j1 - j0);
  const int threads = 256;
  const int64_t blocks = (total + threads - 1) / threads;
  const unsigned grid = (unsigned)(blocks < 148 * 64 ? blocks : 148 * 64);
  const PhiloxKeys K = make_keys(seed);
#define SK_FILL(D, T) sk_fill_s_kernel<D, T><<<grid, threads, 0, stream>>>(K, i0, i1, j0, j1, q0, nq, (T*)out, ld)
  if (dist == 0) { if (dtype == 0) SK_FILL(0, double); else SK_FILL(0, float); }
  else if (dist == 1) { if (dtype == 0) SK_FILL(1, double); else SK_FILL(1, float); }
  else if (dist == 3) { if (dtype == 0) SK_FILL(3, double); else SK_FILL(3, float); }
  else { if (dtype == 0) SK_FILL(2, double); else SK_FILL(2, float); }
#undef SK_FILL
  return cudaGetLastError();
}

// Distinct rows of rowidx[p0, p1) (plan-time sampling for Algorithm 4): each entry sets its row's
// bit in a zeroed bitmap; entries that find the bit clear are counted (warp-aggregated).
__global__ void sk_distinct_rows_kernel(const int32_t* __restrict__ rowidx, int64_t p0, int64_t p1,
                                        uint32_t* __restrict__ bitmap, unsigned long long* __restrict__ count) {
  unsigned long long mine = 0;
  for (int64_t p = p0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < p1; p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r = (uint32_t)__ldg(rowidx + p), bit = 1u << (r & 31);
    mine += (atomicOr(bitmap + (r >> 5), bit) & bit) ? 0 : 1;
  }
  for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xFFFFFFFFu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(count, mine);
}

cudaError_t launch_distinct_rows(const int32_t* rowidx, int64_t p0, int64_t p1, uint32_t* bitmap,
                                 unsigned long long* count, cudaStream_t stream) {
  if (p1 <= p0) return cudaSuccess;
  const int threads = 256;
  int64_t blocks = (p1 - p0 + threads - 1) / threads;
  if (blocks > 148 * 8) blocks = 148 * 8;
  sk_distinct_rows_kernel<<<(unsigned)blocks, threads, 0, stream>>>(rowidx, p0, p1, bitmap, count);
  return cudaGetLastError();
}

cudaError_t launch_validate_rows(const int32_t* rowidx, int64_t nnz, int64_t m, int* flag,
                                 cudaStream_t stream) {
  if (nnz == 0) return cudaSuccess;
  const int threads = 256;
  int64_t blocks = (nnz + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  sk_validate_rows_kernel<<<(unsigned)blocks, threads, 0, stream>>>(rowidx, nnz, m, flag);
  return cudaGetLastError();
}

}  // namespace sk
