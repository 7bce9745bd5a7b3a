/*
 * sketch.h -- C ABI of libsketch: the B200-native on-the-fly-RNG sketch  Â = S·A.
 *
 * The operation (arXiv 2310.15419, Eq. `goal`): A is a tall sparse
 * m x n matrix in CSC form ("we take CSC as our default sparse matrix
 * format"), S is a d x m matrix with i.i.d. entries that is NEVER stored: every entry
 * S[i, j] is regenerated on the fly from a counter-based RNG keyed by its row/column
 * indices (§4.2 "Counter Based RNG"), and  Â = S·A  (d x n, dense).
 * Entry distributions are the paper's three: ±1 (Rademacher),
 * uniform over (-1, 1), and mean-zero Gaussian.
 *
 * Entry definition (readings R1-R5; bit-exact, independent of tiling, launch
 * shape and GPU count -- the reproducibility of PAPER.md:511):
 *   block(q, j) = Philox4x32-10(counter = (q, 0, j mod 2^32, j div 2^32),
 *                               key     = (seed mod 2^32, seed div 2^32))  -> x[0..3]
 *   SK_RADEMACHER : q = i/128, t = (i%128)/32, b = i%32;  S = (bit b of x[t]) ? -1 : +1
 *   SK_UNIFORM    : q = i/2, h = i%2, k = (x[2h]*2^32 + x[2h+1]) >> 11;
 *                   S = (2k + 1 - 2^53) * 2^-53                       (open (-1,1), exact)
 *   SK_GAUSSIAN   : q = i/2, k1 = (x0*2^32+x1)>>11, k2 = (x2*2^32+x3)>>11,
 *                   u1 = (k1+1) 2^-53, u2 = k2 2^-53, rho = sqrt(-2 ln u1),
 *                   th = u2 * fl64(2 pi);  S[2q] = rho cos th, S[2q+1] = rho sin th
 *   SK_UNIFORM24  : q = i/4, t = i%4, k = x[t] >> 8;  S = (2k + 1 - 2^24) * 2^-24
 *                   (a cheaper uniform(-1,1) for 32-bit work, PAPER.md:464;
 *                   4 entries per block, exact in fp32 -- a different S than SK_UNIFORM)
 *   dtype SK_F32  : S32 = round-to-nearest-even(S64); arithmetic in fp32.
 * Here j is the GLOBAL row index of A (row_offset + local row), i the row of Â.
 *
 * Conventions for every entry point:
 *  - Indices are 0-based.  colptr is int64[n+1] (colptr[0] = 0, non-decreasing,
 *    colptr[n] = nnz), rowidx is int32[nnz] with 0 <= rowidx < m.  Rows inside a column
 *    may be unsorted and may repeat; explicit zeros are processed (linearity).
 *  - Non-finite values: a NaN value makes every entry of its column NaN (as NaN * ±1 does).
 *    The SIMT kernels (fp32, uniform, Gaussian) follow IEEE arithmetic for +-Inf too; the
 *    exact ±1 fp64 tensor-core kernel (the default for SK_RADEMACHER + SK_F64) writes NaN to
 *    the whole column when it holds a NaN or an Inf (its digit encoding needs finite values).
 *  - Pointers are DEVICE pointers unless the name starts with h_ (host memory; pinned
 *    host memory is required for overlap but not for correctness).
 *  - out is d x n COLUMN-MAJOR with leading dimension d, and is OVERWRITTEN in full
 *    (beta = 0; empty columns are written as zeros -- Algorithm 1 initialises Â = 0,
 *    PAPER.md:83).  out must not alias any input.
 *  - The caller owns every buffer passed in; they must stay valid until the stream work
 *    that uses them has completed.  A plan references (does not copy) colptr/rowidx.
 *  - stream: a cudaStream_t (NULL = legacy default stream).
 *  - Return value: 0 on success, a negative sk_status code otherwise.  No C++ exception
 *    crosses this boundary.  sketch_error_string() describes a code; after SK_ECUDA,
 *    sketch_last_error_detail() gives the CUDA error text of the calling thread.
 */
#ifndef LIBSKETCH_SKETCH_H
#define LIBSKETCH_SKETCH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* sk_stream_t;           /* == cudaStream_t */

typedef enum { SK_RADEMACHER = 0, SK_UNIFORM = 1, SK_GAUSSIAN = 2, SK_UNIFORM24 = 3 } sk_dist_t;
typedef enum { SK_F64 = 0, SK_F32 = 1 } sk_dtype_t;

typedef enum {
    SK_OK = 0,
    SK_EINVAL = -1,        /* bad argument: NULL with nonzero size, d < 1, m/n < 0, bad enum,
                              d >= 2^31, m >= 2^31 (rowidx is int32), row_offset < 0 */
    SK_ECSC = -2,          /* CSC validation failed (colptr / rowidx out of contract) */
    SK_ENOMEM = -3,        /* device or host allocation failed */
    SK_ECUDA = -4,         /* a CUDA runtime call or kernel launch failed */
    SK_EUNSUPPORTED = -5   /* valid request this build does not implement */
} sk_status;

typedef struct sk_plan_s* sk_plan_t;                /* opaque; owned by the library */

typedef struct {
    int64_t d, m, n, nnz;
    int64_t row_offset;
    int64_t max_col_nnz;       /* longest column */
    int64_t n_items_rad;       /* CTAs of one SK_RADEMACHER apply */
    int64_t n_items_pair;      /* CTAs of one SK_UNIFORM / SK_GAUSSIAN apply */
    int64_t philox_blocks_rad; /* Philox4x32-10 calls of one SK_RADEMACHER apply (Alg. 3 count) */
    int64_t philox_blocks_pair;/* Philox calls of one SK_UNIFORM / SK_GAUSSIAN apply */
    int64_t plan_bytes;        /* device bytes the plan owns */
    int64_t n_items_jki;       /* work items of the Algorithm 4 (jki) path, 0 if not built */
    int64_t jki_nonzero_rows;  /* Σ over 16-column groups of the group's nonzero rows (its RNG work) */
    int64_t n_items_f4_split;  /* fp4 tensor-core items that are halves of a last-wave item split along
                                  K (0: no split; > 0: apply also launches a small zeroing kernel) */
} sk_stats_t;

/*
 * sketch_plan -- validate a CSC matrix and build the launch schedule (work items ordered
 * longest-first) used by sketch_apply.  This is the analogue of the paper's "format
 * conversion" step (timed separately as the paper does).
 * SYNCHRONOUS on `stream`: it reads colptr back to the host and validates rowidx on the
 * device before returning.  m is the number of LOCAL rows; row_offset is the global
 * index of local row 0 (row sharding across GPUs: RNG keys use global rows).
 * Errors: SK_EINVAL, SK_ECSC, SK_ENOMEM, SK_ECUDA.  *plan is NULL on error.
 */
int sketch_plan(sk_plan_t* plan, sk_dtype_t dtype, int64_t d, int64_t m, int64_t n,
                int64_t row_offset, const int64_t* colptr, const int32_t* rowidx,
                int64_t nnz, sk_stream_t stream);

/* sketch_plan_host -- as sketch_plan, but colptr is given in HOST memory (h_colptr; the
 * plan keeps no reference to it) and rowidx is still a device pointer.  Row validation
 * is skipped when validate_rows == 0 (the caller vouches for the rows), which makes the
 * call asynchronous apart from the small schedule upload. */
int sketch_plan_host(sk_plan_t* plan, sk_dtype_t dtype, int64_t d, int64_t m, int64_t n,
                     int64_t row_offset, const int64_t* h_colptr, const int32_t* rowidx,
                     int64_t nnz, int validate_rows, sk_stream_t stream);

/*
 * sketch_apply -- out = S[:, row_offset : row_offset+m] · A  (d x n, column-major, ld = d).
 * vals: nnz values in the plan's dtype (double for SK_F64, float for SK_F32), same order
 * as rowidx.  ASYNCHRONOUS, stream-ordered; plan is read-only (concurrent applies of one
 * plan on different streams are allowed).  Fused kernels: Philox generation, transform,
 * multiply-accumulate, in-CTA reduction and a single store of every Â tile.
 * Errors: SK_EINVAL (bad enum / NULL), SK_ECUDA (launch failure).
 */
int sketch_apply(sk_plan_t plan, uint64_t seed, sk_dist_t dist, const void* vals, void* out,
                 sk_stream_t stream);

/* sketch_apply_csc -- one-shot form of the north-star signature: plan + apply + destroy.
 * Synchronous (planning reads colptr back).  Same semantics as sketch_apply. */
int sketch_apply_csc(uint64_t seed, sk_dist_t dist, sk_dtype_t dtype, int64_t d, int64_t m,
                     int64_t n, int64_t row_offset, const int64_t* colptr,
                     const int32_t* rowidx, int64_t nnz, const void* vals, void* out,
                     sk_stream_t stream);

/*
 * sketch_apply_host -- end-to-end form with HOST buffers: copies A (h_colptr, h_rowidx,
 * h_vals) to the device, plans, applies and copies Â back into h_out (d x n column-major).
 * The column range is processed in `pipeline_chunks` column groups (0 = automatic) so the
 * host->device copy of group g+1 overlaps the kernels of group g and the device->host copy
 * of group g-1.  Device scratch is allocated stream-ordered and freed before returning.
 * Synchronous: returns after h_out is complete.  Errors: as sketch_plan / sketch_apply.
 */
int sketch_apply_host(uint64_t seed, sk_dist_t dist, sk_dtype_t dtype, int64_t d, int64_t m,
                      int64_t n, int64_t row_offset, const int64_t* h_colptr,
                      const int32_t* h_rowidx, const void* h_vals, void* h_out,
                      int pipeline_chunks, sk_stream_t stream);

/*
 * sketch_fill_s -- materialise S[i0:i1, j0:j1] (global indices) into out, column-major
 * with leading dimension ld >= i1 - i0, in dtype (double / float).  Asynchronous.
 * This is the parity anchor for the RNG contract above (bit-exact for ±1 and uniform).
 * Errors: SK_EINVAL (bad range / enum / ld), SK_ECUDA.
 */
int sketch_fill_s(uint64_t seed, sk_dist_t dist, sk_dtype_t dtype, int64_t i0, int64_t i1,
                  int64_t j0, int64_t j1, void* out, int64_t ld, sk_stream_t stream);

/* sketch_plan_stats -- copy the plan's statistics to host memory. Errors: SK_EINVAL. */
int sketch_plan_stats(sk_plan_t plan, sk_stats_t* h_stats);

/* sketch_plan_destroy -- free the plan's device and host memory (after its stream work
 * has completed).  NULL is accepted.  Errors: SK_ECUDA. */
int sketch_plan_destroy(sk_plan_t plan);

/* sketch_error_string -- static text for a status code. */
const char* sketch_error_string(int code);

/* sketch_last_error_detail -- thread-local text of the last CUDA error seen by this thread. */
const char* sketch_last_error_detail(void);

/* sketch_version -- "libsketch <version> sm_100a". */
const char* sketch_version(void);

/*
 * Kernel selection for SK_RADEMACHER with SK_F64 values (process-wide).  All paths compute the
 * same Â within the parity bound (|Â - oracle| <= 1e-12 |S||A|); the tensor-core paths are
 * exact up to the per-column fixed-point rounding of the values (<= 2^-44 |S||A| for
 * SK_PATH_TC_FP4..HYBRID, <= 2^-42 |S||A| for SK_PATH_TC_FP4N) and a single final fp64 rounding.
 * Tensor-core paths need an average of >= 256 nonzeros per column and every column to hold
 * <= 131071 nonzeros (SK_PATH_TC_FP4N: <= 1048575), else the SIMT kernel runs.
 * Default: SK_PATH_TC_FP4, or the SKETCH_RAD_F64_PATH environment variable
 * (fp4 | fp4t | fp4n | int8smem | int8tmem | simt | hybrid).  SK_PATH_TC_FP4N also needs 16-byte aligned
 * rowidx / vals (TMA) and colptr[n] < 2^31 - 512.  Errors: SK_EINVAL for an unknown path.
 */
typedef enum {
    SK_PATH_TC_FP4 = 0,        /* tcgen05 kind::mxf4: ±1 as e2m1, values as 64 signed binary digits */
    SK_PATH_TC_INT8_SMEM = 1,  /* tcgen05 kind::i8: S tiles in smem (MN-major), 8 int8 digit planes */
    SK_PATH_TC_INT8_TMEM = 2,  /* tcgen05 kind::i8: S tiles in TMEM (K-major) */
    SK_PATH_SIMT = 3,          /* FP64 SIMT kernel: one SEL + one DADD per (row, nonzero) */
    SK_PATH_HYBRID = 4,        /* one persistent kernel: int8 tensor-core warps + FP64 SIMT warps
                                  pulling columns from one queue */
    SK_PATH_TC_FP4N = 5,       /* tcgen05 kind::mxf4, S as the N = 256 operand, values as 63 magnitude
                                  digits, TMA-fed persistent kernel */
    SK_PATH_TC_FP4T = 6        /* tcgen05 kind::mxf4 with the S operand written to / read from TMEM */
} sk_rad_f64_path_t;
int sketch_set_rad_f64_path(int path);

/*
 * Kernel selection for SK_RADEMACHER with SK_F32 values (process-wide; both compute Â in fp32
 * within the parity bound 2e-5 |S||A|).  SK_PATH32_SIMT (default): one predicated add per
 * (row, nonzero).  SK_PATH32_TABLE: per 4 nonzeros the CTA tabulates the 16 signed sums
 * ±a_1 ±a_2 ±a_3 ±a_4 and each row adds the one its 4 sign bits select (one table load + one add
 * per 4 entries; sums formed in nonzero order).  Initialised from SKETCH_RAD_F32_PATH = simt | tab.
 * Errors: SK_EINVAL for an unknown path.
 */
typedef enum { SK_PATH32_SIMT = 1, SK_PATH32_TABLE = 0 } sk_rad_f32_path_t;
int sketch_set_rad_f32_path(int path);

/*
 * Kernel selection for SK_UNIFORM / SK_GAUSSIAN (process-wide): Algorithm 3 (kji: S[:, j] regenerated
 * per stored nonzero) or Algorithm 4 (jki: S[:, j] regenerated once per nonzero
 * row of each 16-column group and reused across the row).  The plan builds the
 * jki structure (the group-wise CSR, "format conversion") only when a sample of column groups shows
 * at least 1.8 nonzeros per nonzero row; SK_PAIR_AUTO then uses jki whenever it was built.
 * Initialised from SKETCH_PAIR_PATH = auto | kji | jki.  Errors: SK_EINVAL.
 */
typedef enum { SK_PAIR_AUTO = 0, SK_PAIR_KJI = 1, SK_PAIR_JKI = 2 } sk_pair_path_t;
int sketch_set_pair_path(int path);

/* sketch_plan_host_jki -- as sketch_plan_host, but always builds the jki structure (for
 * measurements and tests of Algorithm 4 on any sparsity pattern).  Same errors. */
int sketch_plan_host_jki(sk_plan_t* plan, sk_dtype_t dtype, int64_t d, int64_t m, int64_t n,
                         int64_t row_offset, const int64_t* h_colptr, const int32_t* rowidx,
                         int64_t nnz, int validate_rows, sk_stream_t stream);

/* sketch_apply_kernel_name -- name of the kernel sketch_apply(plan, *, dist, ...) launches
 * ("" for a NULL plan or bad dist).  Static string, for reporting. */
const char* sketch_apply_kernel_name(sk_plan_t plan, sk_dist_t dist);

#ifdef __cplusplus
}
#endif

#endif /* LIBSKETCH_SKETCH_H */
