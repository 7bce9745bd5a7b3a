// sketch_api.cu -- the C ABI of libsketch (include/sketch.h): argument checking, the plan
// (validation + longest-first work schedule) and the launch of the sm_100a kernels.
//
// The plan is the GPU analogue of the paper's "format conversion" step (PAPER.md:444-445,
// 619-641): the kji kernel needs only the CSC structure ("Algorithm 3 only
// requires standard CSC"), so planning is just validation plus the order in which the
// (column, Â-row tile) work items of Algorithm 1's outer loops are
// handed to CTAs -- the parallelised outer loops of PAPER.md:327-332.
#include <algorithm>
#include <chrono>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/sketch.h"
#include "kernels.h"
#include "philox.cuh"

using sk::Item;

namespace sk {
// One memory pool per device for the library's stream-ordered scratch (jki values / workspace, the
// device copies of sketch_apply_host).  Its release threshold is unlimited: freed blocks stay mapped
// for the next call instead of being returned to the driver at every synchronisation (the default
// pool's threshold 0 re-maps hundreds of MB per call).  The pool holds the high-water mark of the
// scratch in flight at once.
cudaError_t scratch_alloc(void** ptr, size_t bytes, cudaStream_t stream) {
  static std::mutex mu;
  static cudaMemPool_t pools[128] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 128) return cudaErrorInvalidDevice;
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!pools[dev]) {
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      e = cudaMemPoolCreate(&pools[dev], &props);
      if (e != cudaSuccess) { pools[dev] = nullptr; return e; }
      uint64_t keep = UINT64_MAX;
      e = cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
      if (e != cudaSuccess) return e;
    }
    pool = pools[dev];
  }
  return cudaMallocFromPoolAsync(ptr, bytes, pool, stream);
}

cudaError_t set_max_dynamic_smem(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, size_t>> done;   // ((kernel, device), bytes)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  for (auto& d : done)
    if (d.first.first == kernel && d.first.second == dev && d.second >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done.push_back({{kernel, dev}, bytes});
  return e;
}
}  // namespace sk

namespace {

thread_local std::string g_detail;

int cuda_fail(cudaError_t e, const char* what) {
  g_detail = std::string(what) + ": " + cudaGetErrorString(e);
  return SK_ECUDA;
}

#define SK_CUDA(call)                                  \
  do {                                                 \
    cudaError_t e_ = (call);                           \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

bool valid_dist(int d) { return d == SK_RADEMACHER || d == SK_UNIFORM || d == SK_GAUSSIAN || d == SK_UNIFORM24; }
bool valid_dtype(int t) { return t == SK_F64 || t == SK_F32; }
size_t dtype_bytes(int t) { return t == SK_F64 ? 8 : 4; }

constexpr int64_t kMaxD = (int64_t(1) << 31) - 1;
constexpr int kSMs = 148;

// Work schedule for one row-tiling (Rademacher: 1024 rows per warp; uniform/Gaussian: 512).
struct Schedule {
  std::vector<Item> items;
  int64_t philox_blocks = 0;
};

// Schedule of the SIMT kernels over the columns `cols` (all n when null).  colptr: n+1 absolute
// offsets (colptr[0] may be nonzero for column sub-ranges).
Schedule build_schedule(const int64_t* colptr, int64_t n, int64_t d, int rows_per_warp,
                        int blocks_per_nnz_per_warp, const std::vector<int32_t>* cols = nullptr) {
  Schedule S;
  const int64_t nc = cols ? (int64_t)cols->size() : n;
  auto col_at = [&](int64_t i) -> int64_t { return cols ? (*cols)[(size_t)i] : i; };
  const int64_t n_rw = (d + rows_per_warp - 1) / rows_per_warp;  // row-warps covering d
  // Cost of one CTA (warps run in parallel): its per-warp nonzero slice plus a fixed overhead
  // (prologue, reduction, store) of about 30 nonzero-equivalents.  W_d (row-warps per CTA,
  // 1..16) minimises Σ_columns tiles × cost for the matrix as a whole.
  auto cost_of = [&](int64_t L, int64_t WD) {
    const int64_t WK = sk::kWarps / WD;
    return (L + WK - 1) / WK + 30;
  };
  int64_t base = 1;
  double best = 1e300;
  // SKETCH_SCHED_WD (tuning only): force W_d for every column
  static const int64_t force_wd = [] { const char* v = getenv("SKETCH_SCHED_WD"); return v ? atoll(v) : 0; }();
  for (int64_t WD = 1; WD <= std::min<int64_t>(16, n_rw); ++WD) {
    if (force_wd > 0 && WD != std::min<int64_t>(force_wd, std::min<int64_t>(16, n_rw))) continue;
    const int64_t tiles = (n_rw + WD - 1) / WD;
    double tot = 0;
    for (int64_t i = 0; i < nc; ++i) {
      const int64_t k = col_at(i);
      tot += (double)tiles * (double)cost_of(colptr[k + 1] - colptr[k], WD);
    }
    if (tot < best * 0.999) { best = tot; base = WD; }
  }
  // Average load per SM slot with the base shape; a column whose CTAs would each exceed a
  // quarter of it is re-shaped to W_d = 1 (16 warps on its nonzero stream) so the longest
  // CTAs do not set the makespan (column-length skew, e.g. power-law columns).
  const double per_slot = best / kSMs;
  std::vector<std::pair<int64_t, Item>> tmp;
  for (int64_t i = 0; i < nc; ++i) {
    const int64_t k = col_at(i);
    const int64_t L = colptr[k + 1] - colptr[k];
    int64_t WD = base;
    if (force_wd == 0 && WD > 1 && (double)cost_of(L, WD) > 0.25 * per_slot) WD = 1;
    const int64_t tiles = (n_rw + WD - 1) / WD;
    for (int64_t tt = 0; tt < tiles; ++tt) {
      Item it;
      it.col = (int32_t)k;
      it.row0 = (int32_t)(tt * WD * rows_per_warp);
      it.wd = (int32_t)WD;
      it.pad = 0;
      tmp.emplace_back(cost_of(L, WD), it);
    }
    S.philox_blocks += L * tiles * WD * blocks_per_nnz_per_warp;
  }
  std::stable_sort(tmp.begin(), tmp.end(),
                   [](const std::pair<int64_t, Item>& a, const std::pair<int64_t, Item>& b) {
                     return a.first > b.first;
                   });
  S.items.reserve(tmp.size());
  for (auto& pr : tmp) S.items.push_back(pr.second);
  return S;
}

// Tensor-core schedule over the columns `cols`: per column, ceil(d/128) row tiles in groups of <= `per`
// per CTA, longest columns first.
std::vector<sk::TcItem> build_tc_schedule(const int64_t* colptr, int64_t d, int64_t per, const std::vector<int32_t>& cols) {
  const int64_t tiles = (d + 127) / 128;
  const int64_t groups = (tiles + per - 1) / per;
  const int64_t tpg = (tiles + groups - 1) / groups;
  std::vector<std::pair<int64_t, sk::TcItem>> tmp;
  for (int32_t k : cols) {
    const int64_t L = colptr[k + 1] - colptr[k];
    for (int64_t g = 0; g * tpg < tiles; ++g) {
      sk::TcItem it;
      it.col = k;
      it.tile0 = (int32_t)(g * tpg);
      it.ntiles = (int32_t)std::min(tpg, tiles - g * tpg);
      it.pad = 0;
      tmp.emplace_back(L, it);
    }
  }
  std::stable_sort(tmp.begin(), tmp.end(), [](const std::pair<int64_t, sk::TcItem>& a,
                                              const std::pair<int64_t, sk::TcItem>& b) { return a.first > b.first; });
  std::vector<sk::TcItem> out;
  out.reserve(tmp.size());
  for (auto& pr : tmp) out.push_back(pr.second);
  return out;
}

// Kernel used for ±1 with fp64 values (process-wide, read when a plan is built; results agree
// within the parity bound): SK_PATH_TC_FP4 (default: the tensor-core kernel for every column of
// f4_min_column(..) .. kTcMaxColumn nonzeros, the SIMT kernel for the others, concurrently) or
// SK_PATH_SIMT (the SIMT kernel for every column).  Initialised from SKETCH_RAD_F64_PATH = fp4 | simt.
std::atomic<int> g_rad_f64_path{-1};

int rad_f64_path() {
  int v = g_rad_f64_path.load(std::memory_order_relaxed);
  if (v >= 0) return v;
  v = SK_PATH_TC_FP4;
  if (const char* e = getenv("SKETCH_RAD_F64_PATH"))
    if (!strcmp(e, "simt")) v = SK_PATH_SIMT;
  g_rad_f64_path.store(v, std::memory_order_relaxed);
  return v;
}

// Shortest column the tensor-core kernel takes (shorter ones go to the SIMT kernel, whose CTA has
// no TMEM / barrier / pipeline fill and drain to amortise): the measured crossover at d = 2000
// (scripts/f4_threshold_sweep.py, profiles/r02_f4_threshold_sweep.txt, tensor-core / SIMT time):
// persistent kernel 1.08 at L = 768, 0.85 at 1024 -> 896; one CTA per item 1.16 at 1024, 0.94 at
// 1536 -> 1280.  SKETCH_F4_MIN_COL (tuning only) overrides both.
int64_t f4_min_column(bool persistent) {
  static const int64_t v = [] { const char* e = getenv("SKETCH_F4_MIN_COL"); return e ? std::max<int64_t>(1, atoll(e)) : 0; }();
  return v > 0 ? v : (persistent ? 896 : 1280);
}

// Persistent tensor-core kernel (one CTA per SM walking the items; TMEM / barriers / constant rows set
// up once, the next item's column scale computed ahead, its first stage produced before the previous
// item's read-out) whenever there is more than one wave of items: it saves the per-item set-up, scan
// and pipeline fill.  Measured (scripts/gpurun/gpu_r2aj.sh, profiles/r02_f4_persistent_sweep.txt), per-item ->
// persistent: c5 7.234 -> 7.165 ms, its 2-way row shard 3.727 -> 3.635, 8-way 1.088 -> 0.988, 1480
// items of 8192 nonzeros 0.726 -> 0.672; one item per SM (148 x 131071) 1.019 -> 1.025, so a single
// wave keeps one CTA per item.  SKETCH_F4_PERSIST = 0 | 1 forces the choice.
std::atomic<int> g_f4_persist{-2};   // -2: not read yet

bool f4_use_persistent(int64_t n_items) {
  int v = g_f4_persist.load(std::memory_order_relaxed);
  if (v == -2) {
    const char* e = getenv("SKETCH_F4_PERSIST");
    v = e ? (atoi(e) != 0 ? 1 : 0) : -1;
    g_f4_persist.store(v, std::memory_order_relaxed);
  }
  if (v >= 0) return v != 0;
  int W = kSMs, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&W, cudaDevAttrMultiProcessorCount, dev);
  return n_items > W;
}

const char* kernel_name(const sk_plan_s* p, int dist);

// Uniform / Gaussian kernel choice (process-wide): SK_PAIR_AUTO (jki when the plan built it),
// SK_PAIR_KJI, SK_PAIR_JKI.  Initialised from SKETCH_PAIR_PATH = auto | kji | jki.
std::atomic<int> g_pair_path{-1};

int pair_path() {
  int v = g_pair_path.load(std::memory_order_relaxed);
  if (v >= 0) return v;
  v = SK_PAIR_AUTO;
  if (const char* e = getenv("SKETCH_PAIR_PATH")) {
    if (!strcmp(e, "kji")) v = SK_PAIR_KJI;
    else if (!strcmp(e, "jki")) v = SK_PAIR_JKI;
  }
  g_pair_path.store(v, std::memory_order_relaxed);
  return v;
}

}  // namespace

struct sk_plan_s {
  sk_dtype_t dtype;
  int64_t d, m, n, nnz, row_offset, max_col;
  const int64_t* colptr;   // device (caller-owned)
  const int32_t* rowidx;   // device (caller-owned)
  Item* d_items = nullptr; // [rad items | pair items | Gaussian items] (SIMT kernels)
  sk::TcItem* d_f4 = nullptr;       // tensor-core ±1 fp64 schedule (empty unless dtype F64 and path FP4)
  int64_t n_f4 = 0;
  int64_t f4_split_items = 0;       // half items of the K-split last wave
  int64_t f4_cols = 0;              // columns on the tensor-core kernel (the rest: n_rad SIMT items)
  bool f4_persist = false;          // the persistent tensor-core kernel (more than one wave of items)
  int64_t f4_split_begin = 0;       // first item of the K-split tail (n_f4: none)
  // Algorithm 4 (jki) structure: one device block holding items, grp_rows, row_j, row_ent, ent, ent_base
  void* d_jki = nullptr;
  sk::JkiPlanView jki{};
  int64_t jki_rows = 0;             // Σ_groups nonzero rows
  int64_t* owned_colptr = nullptr;  // device copy made by sketch_plan_host
  // All schedules live in ONE device block uploaded by one copy.
  void* d_stage = nullptr;
  std::vector<unsigned char> h_stage;   // host image of d_stage (kept until uploaded)
  size_t off_items = 0, off_f4 = 0;
  int64_t n_rad = 0, n_pair = 0, n_gauss = 0;
  int64_t philox_rad = 0, philox_pair = 0;
};

namespace {

// Algorithm 4 structure ("A will need to be first partitioned into vertical
// blocks, and within each block, the entries will be stored in CSR format"), the paper's "format
// conversion".  Blocks are b_n = jki_block_cols(dtype) consecutive
// columns (all n when n <= b_n: every needed S entry is generated once).  The exact number of
// distinct rows per block (device row bitmap) decides whether the Philox work saved pays for the
// shared-memory scatter of every entry.  Measured (r2 reuse sweep, d = 2000, n = 1000 columns of 1000
// nonzeros drawn from R rows, profiles/r02_jki_reuse_sweep.jsonl): Algorithm 4 costs
// ~2.2 ms per 1e6 entries (f32 ~1.4: the scatter is bound by shared-memory bandwidth, 24 B per row x
// entry in fp64) plus 4.3e-6 ms per nonzero row (uniform; Gaussian 6.6e-6; f32 4.6e-6 / 6.8e-6),
// Algorithm 3 2.72 ms per 1e6 entries (uniform; Gaussian 4.94; f32 2.77 / 5.61).  Algorithm 4 is
// chosen when nonzero rows <= kJRowsPerNnz[dtype][dist] x nnz:
//   f64: uniform 0.10 (reuse >= 10), Gaussian 0.40 (reuse >= 2.5);
//   f32: uniform 0.30, Gaussian 0.55.
// The structure is built (unless forced) only when the dtype's Gaussian bar (the loosest) holds.
constexpr double kJRowsPerNnz[2][2] = {{0.10, 0.40}, {0.30, 0.55}};   // [f64, f32][uniform, Gaussian]
double jki_bar(int dtype, int dist) { return kJRowsPerNnz[dtype == SK_F64 ? 0 : 1][dist == SK_GAUSSIAN ? 1 : 0]; }
constexpr double kJScatter = 0.4;   // batch cost in nonzero-row units: rows + kJScatter entries

int build_jki(sk_plan_s* p, const int64_t* h_colptr, bool force, cudaStream_t stream) {
  const int64_t n = p->n, nnz = p->nnz, m = p->m, d = p->d;
  if (n == 0 || nnz == 0) return SK_OK;
  auto unsupported = [&](const char* why) -> int {
    if (!force) return SK_OK;
    g_detail = why;
    return (int)SK_EUNSUPPORTED;
  };
  if (nnz >= (int64_t(1) << 32) - 1) return unsupported("jki: nnz >= 2^32 (32-bit value indices)");
  if (m > (int64_t(1) << 27)) return unsupported("jki: m > 2^27 (host row counters)");
  const int64_t bn = sk::jki_block_cols((int)p->dtype), NB = (n + bn - 1) / bn;
  if (NB > 32767) return unsupported("jki: more than 32767 column blocks");
  const int64_t base = h_colptr[0];
  auto block_range = [&](int64_t b) {   // entries of block b, relative to base
    const int64_t c0 = b * bn, c1 = std::min<int64_t>(n, c0 + bn);
    return std::make_pair(h_colptr[c0] - base, h_colptr[c1] - base);
  };
  // (1) exact distinct rows per block on the device: one row bitmap, one pass per block.  Unless
  // forced, a first pass over at most 2^23 entries (a column prefix of the blocks) skips matrices whose
  // reuse cannot reach the bar: extrapolating its repeats linearly over the whole block must reach it.
  std::vector<unsigned long long> brows((size_t)NB, 0);
  if (!force) {
    int64_t tot_s = 0, tot_all = 0;
    std::vector<std::pair<int64_t, int64_t>> pre;
    for (int64_t b = 0; b < NB; ++b) {
      const auto pr = block_range(b);
      const int64_t take = std::min<int64_t>(pr.second - pr.first, std::max<int64_t>(1, (int64_t(1) << 23) / NB));
      pre.emplace_back(pr.first, pr.first + take);
      tot_s += take;
      tot_all += pr.second - pr.first;
    }
    if (tot_s < tot_all) {
      const size_t words = (size_t)((m + 31) / 32);
      uint32_t* bitmap = nullptr;
      unsigned long long* cnt = nullptr;
      std::vector<unsigned long long> h((size_t)NB, 0);
      SK_CUDA(sk::scratch_alloc((void**)&bitmap, std::max<size_t>(words, 1) * 4, stream));
      cudaError_t e = sk::scratch_alloc((void**)&cnt, (size_t)NB * 8, stream);
      if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, (size_t)NB * 8, stream);
      for (int64_t b = 0; b < NB && e == cudaSuccess; ++b) {
        e = cudaMemsetAsync(bitmap, 0, std::max<size_t>(words, 1) * 4, stream);
        if (e == cudaSuccess) e = sk::launch_distinct_rows(p->rowidx, pre[(size_t)b].first, pre[(size_t)b].second, bitmap, cnt + b, stream);
      }
      if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), cnt, (size_t)NB * 8, cudaMemcpyDeviceToHost, stream);
      cudaFreeAsync(bitmap, stream);
      if (cnt) cudaFreeAsync(cnt, stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
      if (e != cudaSuccess) return cuda_fail(e, "jki sample");
      int64_t rows_s = 0;
      for (auto r : h) rows_s += (int64_t)r;
      const double repeats = (double)(tot_s - rows_s) * (double)tot_all / (double)std::max<int64_t>(tot_s, 1);
      if ((double)tot_all - repeats > jki_bar((int)p->dtype, SK_GAUSSIAN) * (double)tot_all) return SK_OK;
    }
  }
  {
    const size_t words = (size_t)((m + 31) / 32);
    uint32_t* bitmap = nullptr;
    unsigned long long* cnt = nullptr;
    SK_CUDA(sk::scratch_alloc((void**)&bitmap, std::max<size_t>(words, 1) * 4, stream));
    cudaError_t e = sk::scratch_alloc((void**)&cnt, (size_t)NB * 8, stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, (size_t)NB * 8, stream);
    for (int64_t b = 0; b < NB && e == cudaSuccess; ++b) {
      const auto pr = block_range(b);
      e = cudaMemsetAsync(bitmap, 0, std::max<size_t>(words, 1) * 4, stream);
      if (e == cudaSuccess) e = sk::launch_distinct_rows(p->rowidx, pr.first, pr.second, bitmap, cnt + b, stream);
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(brows.data(), cnt, (size_t)NB * 8, cudaMemcpyDeviceToHost, stream);
    cudaFreeAsync(bitmap, stream);
    if (cnt) cudaFreeAsync(cnt, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return cuda_fail(e, "jki distinct rows");
  }
  int64_t rows_total = 0;
  for (auto r : brows) rows_total += (int64_t)r;
  if (!force && !((double)rows_total <= jki_bar((int)p->dtype, SK_GAUSSIAN) * (double)nnz)) return SK_OK;

  // (2) host CSR of every block: counting sort by row, stable in storage (= column) order
  std::vector<int32_t> rows((size_t)nnz);
  SK_CUDA(cudaMemcpyAsync(rows.data(), p->rowidx, (size_t)nnz * 4, cudaMemcpyDeviceToHost, stream));
  SK_CUDA(cudaStreamSynchronize(stream));
  std::vector<int32_t> cnt((size_t)m, 0), touched, row_j;
  std::vector<std::pair<uint32_t, uint32_t>> tmp;   // (value index, column within block) in row order
  std::vector<uint2> ent;
  ent.reserve((size_t)nnz);
  std::vector<sk::JBatch> batches;
  std::vector<uint16_t> own;
  std::vector<double> bcost;                        // per batch: rows + kJScatter entries
  std::vector<int64_t> blk_b0{0};                   // batches of block b: [blk_b0[b], blk_b0[b + 1])
  for (int64_t b = 0; b < NB; ++b) {
    const int64_t c0 = b * bn, c1 = std::min<int64_t>(n, c0 + bn);
    touched.clear();
    for (int64_t q = h_colptr[c0] - base; q < h_colptr[c1] - base; ++q) {
      const int32_t j = rows[(size_t)q];
      if (cnt[(size_t)j]++ == 0) touched.push_back(j);
    }
    std::sort(touched.begin(), touched.end());
    int64_t run = 0;
    for (int32_t j : touched) { const int32_t c = cnt[(size_t)j]; cnt[(size_t)j] = (int32_t)run; run += c; }
    tmp.assign((size_t)run, {0u, 0u});
    for (int64_t k = c0; k < c1; ++k)
      for (int64_t q = h_colptr[k] - base; q < h_colptr[k + 1] - base; ++q)
        tmp[(size_t)cnt[(size_t)rows[(size_t)q]]++] = {(uint32_t)(q + base), (uint32_t)(k - c0)};
    // rows in ascending order; a row's entries in [end of previous row, cnt[j]) after the scatter
    int64_t e0 = 0;
    sk::JBatch cur{};
    auto close = [&]() {
      if (cur.nrows == 0) return;
      // entries of the batch reordered by owner (column mod kJOwners), stable
      const size_t first = (size_t)cur.ent0;
      uint16_t off[sk::kJOwners + 1] = {0};
      for (int32_t e = 0; e < cur.nent; ++e) ++off[(ent[first + e].y & 0xFFFFu) % sk::kJOwners + 1];
      for (int h = 0; h < sk::kJOwners; ++h) off[h + 1] = (uint16_t)(off[h + 1] + off[h]);
      std::vector<uint2> sorted((size_t)cur.nent);
      uint16_t pos[sk::kJOwners];
      std::copy(off, off + sk::kJOwners, pos);
      for (int32_t e = 0; e < cur.nent; ++e) sorted[pos[(ent[first + e].y & 0xFFFFu) % sk::kJOwners]++] = ent[first + e];
      std::copy(sorted.begin(), sorted.end(), ent.begin() + (int64_t)first);
      own.insert(own.end(), off, off + sk::kJOwners + 1);
      own.resize(own.size() + (sk::kJOwnStride - sk::kJOwners - 1), 0);
      bcost.push_back((double)cur.nrows + kJScatter * (double)cur.nent);
      batches.push_back(cur);
      cur = sk::JBatch{};
    };
    for (int32_t j : touched) {
      int64_t e1 = cnt[(size_t)j];
      while (e0 < e1) {   // a row with more than kJBatchEnt entries is cut into several row occurrences
        const int64_t take = std::min<int64_t>(e1 - e0, sk::kJBatchEnt);
        if (cur.nrows > 0 && (cur.nrows == sk::kJBatch || cur.nent + take > sk::kJBatchEnt)) close();
        if (cur.nrows == 0) { cur.ent0 = (int64_t)ent.size(); cur.row0 = (int32_t)row_j.size(); cur.block = (int16_t)b; }
        for (int64_t e = e0; e < e0 + take; ++e)
          ent.push_back(make_uint2(tmp[(size_t)e].first, tmp[(size_t)e].second | ((uint32_t)cur.nrows << 16)));
        row_j.push_back(j);
        cur.nrows = (int16_t)(cur.nrows + 1);
        cur.nent += (int32_t)take;
        e0 += take;
      }
    }
    close();
    for (int32_t j : touched) cnt[(size_t)j] = 0;
    blk_b0.push_back((int64_t)batches.size());
  }
  if (row_j.size() >= (size_t)INT32_MAX) return unsupported("jki: too many nonzero rows");
  // (3) work items: T tiles x P_b parts of each block's batches (equal cost), P chosen so the item
  // count fills whole waves of the SMs (one 200 KB CTA per SM) with >= 4 waves
  const int64_t T = (d + sk::kJRows - 1) / sk::kJRows;
  std::vector<double> blk_cost((size_t)NB, 0.0);
  double tot = 0;
  for (int64_t b = 0; b < NB; ++b)
    for (int64_t t = blk_b0[b]; t < blk_b0[b + 1]; ++t) { blk_cost[(size_t)b] += bcost[(size_t)t]; tot += bcost[(size_t)t]; }
  int W = kSMs, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&W, cudaDevAttrMultiProcessorCount, dev);
  auto parts_for = [&](int64_t ptot) {
    std::vector<int64_t> pb((size_t)NB);
    for (int64_t b = 0; b < NB; ++b) {
      const int64_t nb = blk_b0[b + 1] - blk_b0[b];
      const int64_t want = (int64_t)std::llround((double)ptot * blk_cost[(size_t)b] / std::max(tot, 1.0));
      pb[(size_t)b] = std::max<int64_t>(1, std::min<int64_t>(want, nb));
    }
    return pb;
  };
  const int64_t pmin = std::max<int64_t>(1, (4 * W + T - 1) / T);
  std::vector<int64_t> best_pb;
  double best_eff = -1;
  for (int64_t ptot = pmin; ptot < pmin + 12; ++ptot) {
    auto pb = parts_for(ptot);
    int64_t items = 0;
    for (auto x : pb) items += T * x;
    const double eff = (double)items / (double)(((items + W - 1) / W) * W);
    if (eff > best_eff + 1e-3) { best_eff = eff; best_pb = pb; }
  }
  std::vector<sk::JItem> items;
  std::vector<int32_t> blk_slot{0};
  int64_t slots = 0;
  for (int64_t b = 0; b < NB; ++b) {
    // part boundaries at equal cost (a block may end up with fewer parts than planned)
    std::vector<int64_t> cut{blk_b0[b]};
    double acc = 0;
    const double target = blk_cost[(size_t)b] / (double)best_pb[(size_t)b];
    for (int64_t t = blk_b0[b]; t < blk_b0[b + 1] && (int64_t)cut.size() < best_pb[(size_t)b]; ++t) {
      acc += bcost[(size_t)t];
      if (acc >= target * (double)cut.size() && t + 1 < blk_b0[b + 1]) cut.push_back(t + 1);
    }
    cut.push_back(blk_b0[b + 1]);
    const int64_t P = (int64_t)cut.size() - 1;
    const int64_t s0 = P > 1 ? slots : -1;
    if (P > 1) slots += P;
    blk_slot.push_back((int32_t)slots);
    for (int64_t pt = 0; pt < P; ++pt)
      for (int64_t t = 0; t < T; ++t)
        items.push_back(sk::JItem{(int32_t)t, (int32_t)b, (int32_t)cut[(size_t)pt], (int32_t)cut[(size_t)pt + 1],
                                  P > 1 ? (int32_t)(s0 + pt) : -1});
  }
  // (4) one device block: items | batches | own | row_j | ent_p | ent_desc | blk_slot
  std::vector<uint32_t> ent_p(ent.size()), ent_desc(ent.size());
  for (size_t e = 0; e < ent.size(); ++e) {
    ent_p[e] = ent[e].x;
    ent_desc[e] = sk::jki_desc(ent[e].y & 0xFFFFu, ent[e].y >> 16, (int)p->dtype);
  }
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t b_items = al(items.size() * sizeof(sk::JItem)), b_bat = al(batches.size() * sizeof(sk::JBatch)),
               b_own = al(own.size() * 2), b_rowj = al(row_j.size() * 4), b_ent = al(ent.size() * 4),
               b_slot = al(blk_slot.size() * 4);
  char* blk = nullptr;
  cudaError_t e = cudaMalloc(&blk, b_items + b_bat + b_own + b_rowj + 2 * b_ent + b_slot);
  if (e != cudaSuccess) return e == cudaErrorMemoryAllocation ? SK_ENOMEM : cuda_fail(e, "cudaMalloc(jki)");
  char* c = blk;
  auto put = [&](const void* src, size_t bytes, size_t span) {
    char* dst = c;
    if (bytes && e == cudaSuccess) e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream);
    c += span;
    return dst;
  };
  sk::JkiPlanView J{};
  J.items = reinterpret_cast<const sk::JItem*>(put(items.data(), items.size() * sizeof(sk::JItem), b_items));
  J.batches = reinterpret_cast<const sk::JBatch*>(put(batches.data(), batches.size() * sizeof(sk::JBatch), b_bat));
  J.own = reinterpret_cast<const uint16_t*>(put(own.data(), own.size() * 2, b_own));
  J.row_j = reinterpret_cast<const int32_t*>(put(row_j.data(), row_j.size() * 4, b_rowj));
  J.ent_p = reinterpret_cast<const uint32_t*>(put(ent_p.data(), ent_p.size() * 4, b_ent));
  J.ent_desc = reinterpret_cast<const uint32_t*>(put(ent_desc.data(), ent_desc.size() * 4, b_ent));
  J.blk_slot = reinterpret_cast<const int32_t*>(put(blk_slot.data(), blk_slot.size() * 4, b_slot));
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) { cudaFree(blk); return cuda_fail(e, "upload jki"); }
  J.n_items = (int64_t)items.size();
  J.n = n;
  J.bn = (int32_t)bn;
  J.n_blocks = (int32_t)NB;
  J.n_slots = slots;
  J.n_ent = (int64_t)ent.size();
  p->d_jki = blk;
  p->jki = J;
  p->jki_rows = rows_total;
  return SK_OK;
}

int check_dims(sk_dtype_t dtype, int64_t d, int64_t m, int64_t n, int64_t row_offset) {
  if (!valid_dtype(dtype) || d < 1 || d > kMaxD || m < 0 || m > kMaxD || n < 0 || n > kMaxD ||
      row_offset < 0)
    return SK_EINVAL;
  return SK_OK;
}

int validate_colptr(const int64_t* h, int64_t n, int64_t nnz, bool require_zero_base) {
  if (require_zero_base && h[0] != 0) return SK_ECSC;
  if (h[n] - h[0] != nnz) return SK_ECSC;
  for (int64_t k = 0; k < n; ++k)
    if (h[k + 1] < h[k]) return SK_ECSC;
  return SK_OK;
}

// Last-wave split of the fp4 schedule.  Items cost about the same and the hardware hands them to
// SMs in order, so N items on W SMs take ceil(N / W) item-times; when the last wave is less than
// half full (0 < N mod W < W/2), splitting the last W + N mod W items into two halves along K
// (same rows, half the nonzeros each) turns the final 2 item-times into 1.5.  The halves add into
// Â with one fp64 atomicAdd each onto zeroed rows: 0 + a + b rounds identically in either order,
// so the output stays deterministic.  SKETCH_F4_SPLIT=0 disables it.  Returns the half items.
int64_t split_f4_tail(std::vector<sk::TcItem>& f4, const int64_t* h_colptr) {
  static const bool off = [] { const char* v = getenv("SKETCH_F4_SPLIT"); return v && !strcmp(v, "0"); }();
  int W = kSMs, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&W, cudaDevAttrMultiProcessorCount, dev);
  const int64_t N = (int64_t)f4.size(), r = W > 0 ? N % W : 0;
  if (off || W <= 0 || N <= W || r == 0 || 2 * r >= W) return 0;
  const int64_t first = N - W - r;
  std::vector<sk::TcItem> out(f4.begin(), f4.begin() + first);
  int64_t halves = 0;
  for (int64_t i = first; i < N; ++i) {
    sk::TcItem it = f4[(size_t)i];
    if (h_colptr[it.col + 1] - h_colptr[it.col] >= 128) {   // at least two K-steps
      it.pad = 1; out.push_back(it);
      it.pad = 2; out.push_back(it);
      halves += 2;
    } else {
      out.push_back(it);
    }
  }
  f4.swap(out);
  return halves;
}

// Copy a plan's schedule image to the device on `stream` (one copy); `sync` waits for it and
// drops the host image, otherwise the image stays alive until the plan is destroyed.
int upload_plan(sk_plan_s* p, cudaStream_t stream, bool sync) {
  if (p->h_stage.empty()) return SK_OK;
  cudaError_t e = cudaMemcpyAsync(p->d_stage, p->h_stage.data(), p->h_stage.size(), cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess && sync) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return cuda_fail(e, "upload plan");
  if (sync) std::vector<unsigned char>().swap(p->h_stage);
  return SK_OK;
}

int make_plan(sk_plan_t* out, sk_dtype_t dtype, int64_t d, int64_t m, int64_t n, int64_t row_offset,
              const int64_t* h_colptr, const int64_t* d_colptr, const int32_t* rowidx, int64_t nnz,
              cudaStream_t stream, int jki = 0 /* 0: sample, 1: force, -1: never */,
              bool defer_upload = false /* true: the caller runs upload_plan */) {
  sk_plan_s* p = new (std::nothrow) sk_plan_s();
  if (!p) return SK_ENOMEM;
  p->dtype = dtype; p->d = d; p->m = m; p->n = n; p->nnz = nnz; p->row_offset = row_offset;
  p->colptr = d_colptr; p->rowidx = rowidx;
  p->max_col = 0;
  for (int64_t k = 0; k < n; ++k) p->max_col = std::max(p->max_col, h_colptr[k + 1] - h_colptr[k]);
  static const bool timing = getenv("SKETCH_TIMING") != nullptr;
  const auto tm0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (timing)
      fprintf(stderr, "  make_plan %s: %.3f ms\n", what,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tm0).count());
  };
  // ±1 x fp64: columns with f4_min_column(..) .. kTcMaxColumn nonzeros run on the tensor cores, the
  // others on the SIMT kernel (per column, not per matrix; the two launches run concurrently)
  std::vector<sk::TcItem> f4;
  std::vector<int32_t> simt_cols;
  const bool use_f4 = dtype == SK_F64 && rad_f64_path() == SK_PATH_TC_FP4;
  if (use_f4) {
    std::vector<int32_t> tc_cols;
    auto route = [&](int64_t min_col) {
      tc_cols.clear();
      simt_cols.clear();
      for (int64_t k = 0; k < n; ++k) {
        const int64_t L = h_colptr[k + 1] - h_colptr[k];
        (L >= min_col && L <= sk::kTcMaxColumn ? tc_cols : simt_cols).push_back((int32_t)k);
      }
    };
    // the persistent kernel pays from f4_min_column(true) nonzeros on; with a single wave of items
    // (the per-item kernel) the longer f4_min_column(false)
    route(f4_min_column(true));
    if (!tc_cols.empty()) {
      const int64_t groups = ((d + 127) / 128 + sk::f4_tiles_per_cta() - 1) / sk::f4_tiles_per_cta();
      if (!f4_use_persistent((int64_t)tc_cols.size() * groups)) route(f4_min_column(false));
    }
    if (!tc_cols.empty()) {
      f4 = build_tc_schedule(h_colptr, d, sk::f4_tiles_per_cta(), tc_cols);
      p->f4_split_items = split_f4_tail(f4, h_colptr);
      p->f4_split_begin = (int64_t)f4.size();
      for (size_t i = 0; i < f4.size(); ++i)
        if (f4[i].pad) { p->f4_split_begin = (int64_t)i; break; }
      p->f4_persist = f4_use_persistent((int64_t)f4.size());
    }
    p->f4_cols = (int64_t)tc_cols.size();
  }
  Schedule rad = build_schedule(h_colptr, n, d, sk::kRowsPerWarpRad, sk::kRowsPerWarpRad / 128,
                                use_f4 ? &simt_cols : nullptr);
  Schedule pair = build_schedule(h_colptr, n, d, sk::kRowsPerWarpPair, sk::kRowsPerWarpPair / 2);
  Schedule gauss = build_schedule(h_colptr, n, d, sk::kRowsPerWarpGauss, sk::kRowsPerWarpGauss / 2);
  p->n_rad = (int64_t)rad.items.size();
  p->n_pair = (int64_t)pair.items.size();
  p->n_gauss = (int64_t)gauss.items.size();
  p->philox_rad = rad.philox_blocks;
  p->philox_pair = pair.philox_blocks;
  p->n_f4 = (int64_t)f4.size();
  lap("schedules");
  // one host image of every schedule, 256-byte aligned sections
  {
    const int64_t total = p->n_rad + p->n_pair + p->n_gauss;
    auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
    p->off_items = 0;
    p->off_f4 = up(p->off_items + (size_t)total * sizeof(Item));
    const size_t bytes = up(p->off_f4 + f4.size() * sizeof(sk::TcItem));
    p->h_stage.assign(bytes, 0);
    unsigned char* h = p->h_stage.data();
    size_t o = p->off_items;
    for (const Schedule* sc : {&rad, &pair, &gauss}) {
      if (!sc->items.empty()) std::memcpy(h + o, sc->items.data(), sc->items.size() * sizeof(Item));
      o += sc->items.size() * sizeof(Item);
    }
    if (!f4.empty()) std::memcpy(h + p->off_f4, f4.data(), f4.size() * sizeof(sk::TcItem));
    cudaError_t e = defer_upload ? sk::scratch_alloc(&p->d_stage, bytes > 0 ? bytes : 256, stream)
                                 : cudaMalloc(&p->d_stage, bytes > 0 ? bytes : 256);
    if (e != cudaSuccess) { delete p; return e == cudaErrorMemoryAllocation ? SK_ENOMEM : cuda_fail(e, "cudaMalloc(plan)"); }
    unsigned char* dst = static_cast<unsigned char*>(p->d_stage);
    p->d_items = total > 0 ? reinterpret_cast<Item*>(dst + p->off_items) : nullptr;
    p->d_f4 = f4.empty() ? nullptr : reinterpret_cast<sk::TcItem*>(dst + p->off_f4);
  }
  lap("image + malloc");
  if (jki >= 0) {
    const int rj = build_jki(p, h_colptr, jki > 0, stream);
    if (rj != SK_OK) { cudaFree(p->d_stage); delete p; return rj; }
  }
  lap("jki");
  if (!defer_upload) {
    const int ru = upload_plan(p, stream, true);
    if (ru != SK_OK) { sketch_plan_destroy(p); return ru; }
  }
  lap("upload");
  *out = p;
  return SK_OK;
}

int validate_rows_sync(const int32_t* rowidx, int64_t nnz, int64_t m, cudaStream_t stream) {
  if (nnz == 0) return SK_OK;
  int* flag = nullptr;
  SK_CUDA(sk::scratch_alloc((void**)&flag, sizeof(int), stream));
  int h = 0;
  cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(int), stream);
  if (e == cudaSuccess) e = sk::launch_validate_rows(rowidx, nnz, m, flag, stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, stream);
  cudaFreeAsync(flag, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return cuda_fail(e, "validate rows");
  return h ? SK_ECSC : SK_OK;
}

// Algorithm 4 for this distribution?  SK_PAIR_JKI: whenever the plan built it; SK_PAIR_AUTO: when the
// reuse clears the distribution's bar (build_jki); SK_PAIR_KJI: never.
bool use_jki(const sk_plan_s* p, int dist) {
  if (p->jki.n_items == 0 || (dist != SK_UNIFORM && dist != SK_GAUSSIAN)) return false;
  const int path = pair_path();
  if (path == SK_PAIR_KJI) return false;
  if (path == SK_PAIR_JKI) return true;
  return (double)p->jki_rows <= jki_bar((int)p->dtype, dist) * (double)p->nnz;
}

// A side stream + fork / join events per host thread and device (created once).
struct SidePipe {
  int dev = -1;
  bool ok = false;
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};

SidePipe& side_pipe() {
  thread_local SidePipe sp;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { sp.ok = false; return sp; }
  if (sp.dev != dev) {
    sp = SidePipe();
    sp.ok = cudaStreamCreateWithFlags(&sp.side, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&sp.fork, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&sp.join, cudaEventDisableTiming) == cudaSuccess;
    sp.dev = dev;
  }
  return sp;
}

int apply_items(const sk_plan_s* p, uint64_t seed, sk_dist_t dist, const void* vals, void* out,
                cudaStream_t stream) {
  sk::ApplyArgs a;
  a.colptr = p->colptr;
  a.rowidx = p->rowidx;
  a.vals = vals;
  a.out = out;
  a.items = dist == SK_RADEMACHER ? p->d_items
            : dist == SK_GAUSSIAN ? p->d_items + p->n_rad + p->n_pair : p->d_items + p->n_rad;
  a.n_items = dist == SK_RADEMACHER ? p->n_rad : dist == SK_GAUSSIAN ? p->n_gauss : p->n_pair;
  a.d = p->d;
  a.ld = p->d;
  a.row_offset = p->row_offset;
  a.keys = sk::make_keys(seed);
  cudaError_t e = cudaSuccess;
  if (dist == SK_RADEMACHER) {
    if (p->n_f4 > 0 && p->n_rad > 0) {
      // tensor-core columns and SIMT columns (short or longer than kTcMaxColumn) write disjoint
      // columns of Â: the SIMT kernel runs concurrently on a side stream (it takes a few SMs
      // first; the tensor-core items fill the rest), joined back before returning
      SidePipe& sp = side_pipe();
      e = sp.ok ? cudaEventRecord(sp.fork, stream) : cudaErrorNotReady;
      if (e == cudaSuccess) e = cudaStreamWaitEvent(sp.side, sp.fork, 0);
      if (e == cudaSuccess) e = sk::launch_apply(0, (int)p->dtype, a, sp.side);
      if (e == cudaSuccess) e = cudaEventRecord(sp.join, sp.side);
      if (e == cudaSuccess) e = sk::launch_apply_rad_f4(a, p->d_f4, p->n_f4, p->f4_split_begin, p->f4_persist, stream);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(stream, sp.join, 0);
    } else if (p->n_f4 > 0) {
      e = sk::launch_apply_rad_f4(a, p->d_f4, p->n_f4, p->f4_split_begin, p->f4_persist, stream);
    } else {
      e = sk::launch_apply(0, (int)p->dtype, a, stream);
    }
    // fp32 "T - 2P" sums: columns holding a NaN / Inf rewritten with the IEEE result (a scan of the values)
    if (e == cudaSuccess && p->dtype == SK_F32 && p->n_rad > 0) e = sk::launch_rad_ieee_fixup(1, a, p->n, stream);
  } else if (use_jki(p, dist)) {
    e = sk::launch_apply_jki((int)dist, (int)p->dtype, a, p->jki, stream);
  } else {
    e = sk::launch_apply((int)dist, (int)p->dtype, a, stream);
  }
  if (e != cudaSuccess) return cuda_fail(e, "launch apply");
  return SK_OK;
}

const char* kernel_name(const sk_plan_s* p, int dist) {
  if (dist == SK_RADEMACHER) {
    if (p->dtype == SK_F32) return "sk_rad_kernel<float>";
    if (p->n_f4 > 0 && p->f4_persist)
      return p->n_rad > 0 ? "sk_rad_f4p_kernel (tcgen05 kind::mxf4, persistent) + sk_rad_kernel<double>"
                          : "sk_rad_f4p_kernel (tcgen05 kind::mxf4, persistent)";
    if (p->n_f4 > 0) return p->n_rad > 0 ? "sk_rad_f4_kernel (tcgen05 kind::mxf4) + sk_rad_kernel<double>"
                                         : "sk_rad_f4_kernel (tcgen05 kind::mxf4)";
    return "sk_rad_kernel<double>";
  }
  const bool f64 = p->dtype == SK_F64;
  if (use_jki(p, dist)) {
    if (dist == SK_UNIFORM) return f64 ? "sk_jki_kernel<uniform, double> (Algorithm 4)" : "sk_jki_kernel<uniform, float> (Algorithm 4)";
    return f64 ? "sk_jki_kernel<gaussian, double> (Algorithm 4)" : "sk_jki_kernel<gaussian, float> (Algorithm 4)";
  }
  if (dist == SK_UNIFORM) return f64 ? "sk_pair_kernel<uniform, double>" : "sk_pair_kernel<uniform, float>";
  if (dist == SK_UNIFORM24) return f64 ? "sk_pair_kernel<uniform24, double>" : "sk_pair_kernel<uniform24, float>";
  return f64 ? "sk_pair_kernel<gaussian, double>" : "sk_pair_kernel<gaussian, float>";
}

}  // namespace

extern "C" {

int sketch_plan(sk_plan_t* plan, sk_dtype_t dtype, int64_t d, int64_t m, int64_t n,
                int64_t row_offset, const int64_t* colptr, const int32_t* rowidx, int64_t nnz,
                sk_stream_t stream_) {
  if (!plan) return SK_EINVAL;
  *plan = nullptr;
  int rc = check_dims(dtype, d, m, n, row_offset);
  if (rc) return rc;
  if (nnz < 0 || !colptr || (nnz > 0 && !rowidx)) return SK_EINVAL;
  cudaStream_t stream = (cudaStream_t)stream_;
  std::vector<int64_t> h((size_t)n + 1);
  static const bool timing = getenv("SKETCH_TIMING") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
  };
  const auto t0 = now();
  SK_CUDA(cudaMemcpyAsync(h.data(), colptr, (size_t)(n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
  SK_CUDA(cudaStreamSynchronize(stream));
  const auto t1 = now();
  rc = validate_colptr(h.data(), n, nnz, true);
  if (rc) return rc;
  rc = validate_rows_sync(rowidx, nnz, m, stream);
  if (rc) return rc;
  const auto t2 = now();
  rc = make_plan(plan, dtype, d, m, n, row_offset, h.data(), colptr, rowidx, nnz, stream);
  if (timing)
    fprintf(stderr, "sketch_plan: colptr D2H %.3f ms, validation %.3f ms, make_plan %.3f ms\n", ms(t0, t1), ms(t1, t2),
            ms(t2, now()));
  return rc;
}

int sketch_plan_host(sk_plan_t* plan, sk_dtype_t dtype, int64_t d, int64_t m, int64_t n,
                     int64_t row_offset, const int64_t* h_colptr, const int32_t* rowidx,
                     int64_t nnz, int validate_rows, sk_stream_t stream_) {
  if (!plan) return SK_EINVAL;
  *plan = nullptr;
  int rc = check_dims(dtype, d, m, n, row_offset);
  if (rc) return rc;
  if (nnz < 0 || !h_colptr || (nnz > 0 && !rowidx)) return SK_EINVAL;
  rc = validate_colptr(h_colptr, n, nnz, true);
  if (rc) return rc;
  cudaStream_t stream = (cudaStream_t)stream_;
  if (validate_rows) {
    rc = validate_rows_sync(rowidx, nnz, m, stream);
    if (rc) return rc;
  }
  int64_t* dc = nullptr;
  SK_CUDA(cudaMalloc(&dc, (size_t)(n + 1) * sizeof(int64_t)));
  cudaError_t e = cudaMemcpyAsync(dc, h_colptr, (size_t)(n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, stream);
  if (e != cudaSuccess) { cudaFree(dc); return cuda_fail(e, "upload colptr"); }
  rc = make_plan(plan, dtype, d, m, n, row_offset, h_colptr, dc, rowidx, nnz, stream);
  if (rc) { cudaFree(dc); return rc; }
  (*plan)->owned_colptr = dc;
  return SK_OK;
}

int sketch_plan_host_jki(sk_plan_t* plan, sk_dtype_t dtype, int64_t d, int64_t m, int64_t n,
                         int64_t row_offset, const int64_t* h_colptr, const int32_t* rowidx,
                         int64_t nnz, int validate_rows, sk_stream_t stream_) {
  if (!plan) return SK_EINVAL;
  *plan = nullptr;
  int rc = check_dims(dtype, d, m, n, row_offset);
  if (rc) return rc;
  if (nnz < 0 || !h_colptr || (nnz > 0 && !rowidx)) return SK_EINVAL;
  rc = validate_colptr(h_colptr, n, nnz, true);
  if (rc) return rc;
  cudaStream_t stream = (cudaStream_t)stream_;
  if (validate_rows) {
    rc = validate_rows_sync(rowidx, nnz, m, stream);
    if (rc) return rc;
  }
  int64_t* dc = nullptr;
  SK_CUDA(cudaMalloc(&dc, (size_t)(n + 1) * sizeof(int64_t)));
  cudaError_t e = cudaMemcpyAsync(dc, h_colptr, (size_t)(n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, stream);
  if (e != cudaSuccess) { cudaFree(dc); return cuda_fail(e, "upload colptr"); }
  rc = make_plan(plan, dtype, d, m, n, row_offset, h_colptr, dc, rowidx, nnz, stream, 1);
  if (rc) { cudaFree(dc); return rc; }
  (*plan)->owned_colptr = dc;
  return SK_OK;
}

int sketch_set_pair_path(int path) {
  if (path < SK_PAIR_AUTO || path > SK_PAIR_JKI) return SK_EINVAL;
  g_pair_path.store(path, std::memory_order_relaxed);
  return SK_OK;
}

int sketch_apply(sk_plan_t plan, uint64_t seed, sk_dist_t dist, const void* vals, void* out,
                 sk_stream_t stream) {
  if (!plan || !valid_dist(dist)) return SK_EINVAL;
  if (plan->n == 0) return SK_OK;                  // nothing to write
  if (!out || (plan->nnz > 0 && !vals)) return SK_EINVAL;
  return apply_items(plan, seed, dist, vals, out, (cudaStream_t)stream);
}

int sketch_apply_csc(uint64_t seed, sk_dist_t dist, sk_dtype_t dtype, int64_t d, int64_t m,
                     int64_t n, int64_t row_offset, const int64_t* colptr, const int32_t* rowidx,
                     int64_t nnz, const void* vals, void* out, sk_stream_t stream) {
  if (!valid_dist(dist)) return SK_EINVAL;
  sk_plan_t p = nullptr;
  int rc = sketch_plan(&p, dtype, d, m, n, row_offset, colptr, rowidx, nnz, stream);
  if (rc) return rc;
  rc = sketch_apply(p, seed, dist, vals, out, stream);
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  int rc2 = sketch_plan_destroy(p);
  if (rc) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "sketch_apply_csc sync");
  return rc2;
}

int sketch_apply_host(uint64_t seed, sk_dist_t dist, sk_dtype_t dtype, int64_t d, int64_t m,
                      int64_t n, int64_t row_offset, const int64_t* h_colptr,
                      const int32_t* h_rowidx, const void* h_vals, void* h_out,
                      int pipeline_chunks, sk_stream_t stream_) {
  if (!valid_dist(dist)) return SK_EINVAL;
  int rc = check_dims(dtype, d, m, n, row_offset);
  if (rc) return rc;
  if (!h_colptr || !h_out) return SK_EINVAL;
  const int64_t nnz = h_colptr[n];
  if (nnz > 0 && (!h_rowidx || !h_vals)) return SK_EINVAL;
  rc = validate_colptr(h_colptr, n, nnz, true);
  if (rc) return rc;
  cudaStream_t stream = (cudaStream_t)stream_;
  const size_t w = dtype_bytes(dtype);

  // Column groups by nnz; group g+1's upload overlaps group g's kernels.  Group sizes shrink
  // geometrically (ratio SKETCH_HOST_RATIO, default 0.84 ~ compute / upload time per byte on c5) so
  // the previous group's kernels finish about when the next group lands, and the compute left
  // after the last upload (the end-to-end tail) is only the small last group's.
  int G = pipeline_chunks > 0 ? pipeline_chunks : (int)std::min<int64_t>(10, std::max<int64_t>(1, nnz / (1 << 21)));
  G = (int)std::max<int64_t>(1, std::min<int64_t>(G, n));
  std::vector<int64_t> cb((size_t)G + 1, 0);
  {
    std::vector<double> wsum((size_t)G + 1, 0.0);
    static const double ratio = [] { const char* v = getenv("SKETCH_HOST_RATIO"); const double r = v ? atof(v) : 0.84;
                                     return r > 0.1 && r <= 1.0 ? r : 0.84; }();
    double wg = 1.0;
    for (int g = 0; g < G; ++g, wg *= ratio) wsum[g + 1] = wsum[g] + wg;
    int64_t k = 0;
    for (int g = 1; g < G; ++g) {
      const int64_t target = (int64_t)((double)nnz * wsum[g] / wsum[G]);
      while (k < n && h_colptr[k] < target) ++k;
      cb[g] = std::max(cb[g - 1], k);
    }
    cb[G] = n;
  }

  // Streams and events are per host thread and device, created once and reused (their creation
  // and destruction cost more than the copy / kernel overlap wins on small calls).  The call is
  // synchronous, so reuse across calls is safe.
  struct HostPipe {
    int dev = -1;
    cudaStream_t h2d = nullptr, d2h = nullptr, comp2 = nullptr;
    std::vector<cudaEvent_t> ev;
  };
  thread_local HostPipe hp;
  cudaError_t e = cudaSuccess;
  const char* what = "";
#define SK_STEP(call) do { if (e == cudaSuccess) { e = (call); if (e != cudaSuccess) what = #call; } } while (0)
  {
    int dev = 0;
    SK_STEP(cudaGetDevice(&dev));
    if (e == cudaSuccess && hp.dev != dev) {
      hp = HostPipe();
      SK_STEP(cudaStreamCreateWithFlags(&hp.h2d, cudaStreamNonBlocking));
      SK_STEP(cudaStreamCreateWithFlags(&hp.d2h, cudaStreamNonBlocking));
      SK_STEP(cudaStreamCreateWithFlags(&hp.comp2, cudaStreamNonBlocking));
      if (e == cudaSuccess) hp.dev = dev;
    }
    while (e == cudaSuccess && hp.ev.size() < (size_t)(2 * G + 2)) {
      cudaEvent_t ev;
      SK_STEP(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      if (e == cudaSuccess) hp.ev.push_back(ev);
    }
  }
  if (e != cudaSuccess) return cuda_fail(e, what);
  cudaStream_t h2d = hp.h2d, d2h = hp.d2h, comp2 = hp.comp2;   // comp2: odd groups' kernels
  std::vector<cudaEvent_t> ev_in(hp.ev.begin() + 2, hp.ev.begin() + 2 + G), ev_done(hp.ev.begin() + 2 + G, hp.ev.begin() + 2 + 2 * G);
  cudaEvent_t ev_start = hp.ev[0], ev_end = hp.ev[1];
  int64_t* d_colptr = nullptr;
  int32_t* d_rowidx = nullptr;
  void* d_vals = nullptr;
  void* d_out = nullptr;
  int* d_flag = nullptr;
  int h_flag = 0;
  SK_STEP(sk::scratch_alloc((void**)&d_colptr, (size_t)(n + 1) * 8, stream));
  SK_STEP(sk::scratch_alloc((void**)&d_rowidx, (size_t)std::max<int64_t>(nnz, 1) * 4, stream));
  SK_STEP(sk::scratch_alloc(&d_vals, (size_t)std::max<int64_t>(nnz, 1) * w, stream));
  SK_STEP(sk::scratch_alloc(&d_out, (size_t)std::max<int64_t>(d * n, 1) * w, stream));
  SK_STEP(sk::scratch_alloc((void**)&d_flag, sizeof(int), stream));
  SK_STEP(cudaMemsetAsync(d_flag, 0, sizeof(int), stream));
  // Order on the upload stream: colptr, group 0 of A, the group plans' schedule images, groups
  // 1.. of A.  The plans (host schedules, same kernels as sketch_apply) are built while group 0
  // is in flight; they reference d_colptr + c0 (absolute offsets) and d_rowidx, whose contents
  // they do not read.
  auto upload_group = [&](int g) {
    const int64_t p0 = h_colptr[cb[g]], p1 = h_colptr[cb[g + 1]];
    if (p1 > p0) {
      SK_STEP(cudaMemcpyAsync(d_rowidx + p0, h_rowidx + p0, (size_t)(p1 - p0) * 4, cudaMemcpyHostToDevice, h2d));
      SK_STEP(cudaMemcpyAsync((char*)d_vals + p0 * w, (const char*)h_vals + p0 * w, (size_t)(p1 - p0) * w,
                              cudaMemcpyHostToDevice, h2d));
    }
  };
  static const bool timing = getenv("SKETCH_TIMING") != nullptr;
  // SKETCH_TIMING: timeline of uploads / kernels / downloads (stderr), relative to the start
  std::vector<cudaEvent_t> tev;
  auto tmark = [&](cudaStream_t st) {
    if (!timing) return;
    cudaEvent_t ev;
    if (cudaEventCreate(&ev) == cudaSuccess) { cudaEventRecord(ev, st); tev.push_back(ev); }
  };
  SK_STEP(cudaEventRecord(ev_start, stream));
  SK_STEP(cudaStreamWaitEvent(h2d, ev_start, 0));
  tmark(h2d);
  SK_STEP(cudaMemcpyAsync(d_colptr, h_colptr, (size_t)(n + 1) * 8, cudaMemcpyHostToDevice, h2d));
  upload_group(0);
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<sk_plan_t> plans((size_t)G, nullptr);
  for (int g = 0; g < G && e == cudaSuccess; ++g) {
    const int64_t c0 = cb[g], c1 = cb[g + 1];
    const int rcp = make_plan(&plans[g], dtype, d, m, c1 - c0, row_offset, h_colptr + c0, d_colptr + c0,
                              d_rowidx, h_colptr[c1] - h_colptr[c0], stream, -1, true);
    if (rcp != SK_OK) { e = cudaErrorUnknown; what = "make_plan(group)"; }
  }
  if (timing)
    fprintf(stderr, "apply_host: %d group plans %.3f ms\n", G,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  SK_STEP(cudaEventRecord(ev_end, stream));          // (reused) the plans' stream-ordered allocations
  SK_STEP(cudaStreamWaitEvent(h2d, ev_end, 0));
  for (int g = 0; g < G && e == cudaSuccess; ++g)
    if (plans[g] && upload_plan(plans[g], h2d, false) != SK_OK) { e = cudaErrorUnknown; what = "upload plan"; }
  SK_STEP(cudaEventRecord(ev_in[0], h2d));
  tmark(h2d);
  for (int g = 1; g < G; ++g) {
    upload_group(g);
    SK_STEP(cudaEventRecord(ev_in[g], h2d));
    tmark(h2d);
  }
  // Consecutive groups' kernels alternate between the caller's stream and comp2, so a group's
  // last partial wave of CTAs overlaps the next group's first one.
  SK_STEP(cudaStreamWaitEvent(comp2, ev_start, 0));
  for (int g = 0; g < G; ++g) {
    const int64_t c0 = cb[g], c1 = cb[g + 1];
    const int64_t p0 = h_colptr[c0], p1 = h_colptr[c1];
    cudaStream_t cs = (g & 1) ? comp2 : stream;
    SK_STEP(cudaStreamWaitEvent(cs, ev_in[g], 0));
    if (p1 > p0 && e == cudaSuccess) e = sk::launch_validate_rows(d_rowidx + p0, p1 - p0, m, d_flag, cs);
    if (e == cudaSuccess && c1 > c0) {
      const int rca = apply_items(plans[g], seed, dist, d_vals, (char*)d_out + (size_t)(c0 * d) * w, cs);
      if (rca != SK_OK) { e = cudaErrorLaunchFailure; what = "launch apply"; }
    }
    SK_STEP(cudaEventRecord(ev_done[g], cs));
    tmark(cs);
    SK_STEP(cudaStreamWaitEvent(d2h, ev_done[g], 0));
    if (c1 > c0)
      SK_STEP(cudaMemcpyAsync((char*)h_out + (size_t)(c0 * d) * w, (char*)d_out + (size_t)(c0 * d) * w,
                              (size_t)((c1 - c0) * d) * w, cudaMemcpyDefault, d2h));   // h_out: host or device (UVA)
  }
  SK_STEP(cudaEventRecord(ev_end, d2h));
  tmark(d2h);
  SK_STEP(cudaStreamWaitEvent(stream, ev_end, 0));
  SK_STEP(cudaMemcpyAsync(&h_flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost, stream));
  if (e != cudaSuccess) {
    // A failed step skipped the later ones (including the join of the side streams into `stream`):
    // drain every stream before the scratch is freed and before h_out is handed back.
    cudaStreamSynchronize(h2d);
    cudaStreamSynchronize(comp2);
    cudaStreamSynchronize(d2h);
    cudaStreamSynchronize(stream);
  }
  if (d_colptr) cudaFreeAsync(d_colptr, stream);
  if (d_rowidx) cudaFreeAsync(d_rowidx, stream);
  if (d_vals) cudaFreeAsync(d_vals, stream);
  if (d_out) cudaFreeAsync(d_out, stream);
  if (d_flag) cudaFreeAsync(d_flag, stream);
  cudaError_t es = cudaStreamSynchronize(stream);
  if (e == cudaSuccess && es != cudaSuccess) { e = es; what = "cudaStreamSynchronize"; }
  if (timing && tev.size() == (size_t)(2 * G + 2)) {
    // tev: [start, in 0 .. in G-1, done 0 .. done G-1, end]
    auto at = [&](size_t i) { float ms = 0; cudaEventElapsedTime(&ms, tev[0], tev[i]); return ms; };
    fprintf(stderr, "apply_host timeline (ms):");
    for (int g = 0; g < G; ++g) fprintf(stderr, " [g%d in %.2f done %.2f]", g, at(1 + g), at(1 + G + g));
    fprintf(stderr, " end %.2f\n", at(2 * G + 1));
  }
  for (auto ev : tev) cudaEventDestroy(ev);

  for (auto pl : plans) sketch_plan_destroy(pl);

#undef SK_STEP
  if (e != cudaSuccess) return cuda_fail(e, what);
  return h_flag ? SK_ECSC : SK_OK;
}

int sketch_fill_s(uint64_t seed, sk_dist_t dist, sk_dtype_t dtype, int64_t i0, int64_t i1,
                  int64_t j0, int64_t j1, void* out, int64_t ld, sk_stream_t stream) {
  if (!valid_dist(dist) || !valid_dtype(dtype)) return SK_EINVAL;
  if (i0 < 0 || i1 < i0 || j0 < 0 || j1 < j0 || i1 > kMaxD || ld < (i1 - i0)) return SK_EINVAL;
  if ((i1 > i0 && j1 > j0) && !out) return SK_EINVAL;
  cudaError_t e = sk::launch_fill_s((int)dist, (int)dtype, seed, i0, i1, j0, j1, out, ld, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "launch fill_s");
  return SK_OK;
}

int sketch_plan_stats(sk_plan_t plan, sk_stats_t* h) {
  if (!plan || !h) return SK_EINVAL;
  h->d = plan->d; h->m = plan->m; h->n = plan->n; h->nnz = plan->nnz;
  h->row_offset = plan->row_offset;
  h->max_col_nnz = plan->max_col;
  h->n_items_rad = plan->n_rad;
  h->n_items_pair = plan->n_pair;
  h->philox_blocks_rad = plan->philox_rad;
  h->philox_blocks_pair = plan->philox_pair;
  h->n_items_jki = plan->jki.n_items;
  h->jki_nonzero_rows = plan->jki_rows;
  h->n_items_f4_split = plan->f4_split_items;
  h->n_items_f4 = plan->n_f4;
  h->n_cols_f4 = plan->f4_cols;
  h->f4_persistent = plan->f4_persist ? 1 : 0;
  h->jki_block_cols = plan->jki.n_items > 0 ? plan->jki.bn : 0;
  h->plan_bytes = (plan->n_rad + plan->n_pair + plan->n_gauss) * (int64_t)sizeof(Item) +
                  plan->n_f4 * (int64_t)sizeof(sk::TcItem) + (plan->owned_colptr ? (plan->n + 1) * 8 : 0);
  return SK_OK;
}

int sketch_plan_destroy(sk_plan_t plan) {
  if (!plan) return SK_OK;
  cudaError_t e = cudaSuccess;
  if (plan->d_stage) e = cudaFree(plan->d_stage);
  if (plan->owned_colptr) { cudaError_t e2 = cudaFree(plan->owned_colptr); if (e == cudaSuccess) e = e2; }
  if (plan->d_jki) { cudaError_t e2 = cudaFree(plan->d_jki); if (e == cudaSuccess) e = e2; }
  delete plan;
  if (e != cudaSuccess) return cuda_fail(e, "cudaFree(plan)");
  return SK_OK;
}

const char* sketch_error_string(int code) {
  switch (code) {
    case SK_OK: return "ok";
    case SK_EINVAL: return "invalid argument";
    case SK_ECSC: return "CSC validation failed";
    case SK_ENOMEM: return "out of memory";
    case SK_ECUDA: return "CUDA error";
    case SK_EUNSUPPORTED: return "unsupported";
    default: return "unknown status";
  }
}

const char* sketch_last_error_detail(void) { return g_detail.c_str(); }

const char* sketch_version(void) { return "libsketch 0.2.0 sm_100a"; }

int sketch_set_f4_persistent(int mode) {
  if (mode < -1 || mode > 1) return SK_EINVAL;
  g_f4_persist.store(mode, std::memory_order_relaxed);
  return SK_OK;
}

int sketch_set_rad_f64_path(int path) {
  if (path != SK_PATH_TC_FP4 && path != SK_PATH_SIMT) return SK_EINVAL;
  g_rad_f64_path.store(path, std::memory_order_relaxed);
  return SK_OK;
}

const char* sketch_apply_kernel_name(sk_plan_t plan, sk_dist_t dist) {
  if (!plan || !valid_dist(dist)) return "";
  return kernel_name(plan, (int)dist);
}

}  // extern "C"
