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
 *  - Non-finite values follow IEEE arithmetic on every path: a NaN value makes every entry of
 *    its column NaN (as NaN * ±1 does); ±Inf values give ±Inf, or NaN where opposite infinities
 *    meet in one sum.
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
    int64_t jki_nonzero_rows;  /* Σ over the Algorithm 4 column blocks of the block's distinct rows (its
                                  RNG work; = nnzrows(A) when one block holds all n columns) */
    int64_t n_items_f4_split;  /* tensor-core items that are halves of a last-wave item split along K */
    int64_t n_items_f4;        /* CTAs of the tensor-core kernel of one SK_RADEMACHER apply */
    int64_t n_cols_f4;         /* columns on the tensor-core kernel (the others: n_items_rad SIMT CTAs) */
    int64_t jki_block_cols;    /* b_n of the Algorithm 4 column blocks (384 f64, 768 f32), 0 if not built */
    int64_t f4_persistent;     /* 1: the tensor-core columns run on the persistent kernel (more items than
                                  SMs; SKETCH_F4_PERSIST = 0 | 1 forces), 0: one CTA per item */
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
 * sketch_apply -- out = S[:, row_offset : row_offset+m] · A  (d x n, column-major, ld = d): the
 * sketch Â = S A of PAPER.md:21-26 (Eq. `goal`), computed with S regenerated on the fly per the
 * counter-based RNG of PAPER.md:489-492 (§4.2) -- Algorithm 3's kji loops or, when
 * the plan built it, Algorithm 4's row reuse.
 * vals: nnz values in the plan's dtype (double for SK_F64, float for SK_F32), same order
 * as rowidx.  ASYNCHRONOUS, stream-ordered; plan is read-only (concurrent applies of one
 * plan on different streams are allowed).  Fused kernels: Philox generation, transform,
 * multiply-accumulate, in-CTA reduction and a single store of every Â tile.
 * Errors: SK_EINVAL (bad enum / NULL), SK_ECUDA (launch failure).
 */
int sketch_apply(sk_plan_t plan, uint64_t seed, sk_dist_t dist, const void* vals, void* out,
                 sk_stream_t stream);

/* sketch_apply_csc -- one-shot form of the north-star signature: plan + apply + destroy -- the
 * paper's format conversion followed by the multiplication (conversion and compute
 * timed apart; CSC input).  Synchronous (planning reads colptr back).  Same semantics and
 * errors as sketch_plan + sketch_apply. */
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
 * h_out may also be a device pointer (unified addressing): Â then stays on the device, e.g. for
 * the cross-GPU sum of row-shard partials.
 * Synchronous: returns after h_out is complete.  Errors: as sketch_plan / sketch_apply.
 */
int sketch_apply_host(uint64_t seed, sk_dist_t dist, sk_dtype_t dtype, int64_t d, int64_t m,
                      int64_t n, int64_t row_offset, const int64_t* h_colptr,
                      const int32_t* h_rowidx, const void* h_vals, void* h_out,
                      int pipeline_chunks, sk_stream_t stream);

/*
 * sketch_fill_s -- materialise S[i0:i1, j0:j1] (global indices) into out, column-major -- the
 * generator Algorithm 3 calls `get_samples` with the entry definitions above
 * (§4.2) --
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
 * Kernel selection for SK_RADEMACHER with SK_F64 values (process-wide, read when a plan is built).
 * Both compute the same Â within the parity bound |Â - oracle| <= 1e-12 |S||A|.
 *  SK_PATH_TC_FP4 (default): the tcgen05 kind::mxf4 kernel (±1 as e2m1, values as 64 signed binary
 *    digits of a per-column fixed-point scale; exact up to the value rounding <= L 2^-62 max|a| and one
 *    final fp64 rounding) for every column with 896 (1280 when the tensor-core items fill at most
 *    one wave of SMs) .. 131071 nonzeros, and the SIMT kernel,
 *    concurrently on a side stream, for the other columns of the same plan.  A column holding a NaN
 *    or an Inf gets the IEEE result (NaN, or the common sign of its infinite terms), as the SIMT
 *    kernel and the oracle do.
 *  SK_PATH_SIMT: the FP64 SIMT kernel (one SEL + one DADD per (row, nonzero)) for every column.
 * Initialised from SKETCH_RAD_F64_PATH = fp4 | simt.  Errors: SK_EINVAL for an unknown path.
 */
typedef enum {
    SK_PATH_TC_FP4 = 0,
    SK_PATH_SIMT = 3
} sk_rad_f64_path_t;
int sketch_set_rad_f64_path(int path);

/*
 * sketch_set_f4_persistent -- how plans built from now on run their tensor-core columns (process-wide):
 * -1 (default) the persistent kernel (one CTA per SM walking the work items, TMEM / barriers set up
 * once, the next item's column scale computed ahead) when there is more than one wave of tensor-core
 * items (more items than SMs), else one CTA per item; 0 always one CTA per item; 1 always persistent.  Same
 * results either way (the same per-item arithmetic).  Initialised from SKETCH_F4_PERSIST = 0 | 1.
 * Errors: SK_EINVAL for another value.
 */
int sketch_set_f4_persistent(int mode);

/*
 * Kernel selection for SK_UNIFORM / SK_GAUSSIAN (process-wide): Algorithm 3 (kji: S[:, j] regenerated
 * per stored nonzero) or Algorithm 4 (jki: S[:, j] regenerated once per nonzero
 * row of each vertical block of b_n columns -- b_n = 384 fp64 / 768 fp32, i.e. all n columns when
 * they fit -- and reused across the row).  The plan counts the distinct
 * rows of every block exactly (device row bitmap) and builds the jki structure (the blocks' CSR, the
 * "format conversion") when nonzero rows <= 0.40 nnz (fp64; 0.55 fp32).  SK_PAIR_AUTO then uses jki
 * where the measured costs favour it: SK_GAUSSIAN at rows <= 0.40 nnz (fp64) / 0.55
 * (fp32), SK_UNIFORM at rows <= 0.10 nnz (fp64) / 0.30 (fp32) -- the scatter of every entry into the
 * block's shared-memory accumulator costs about as much as generating a uniform S entry;
 * SK_PAIR_JKI uses jki for both whenever it was built (sketch_plan_host_jki always builds it).
 * Initialised from SKETCH_PAIR_PATH = auto | kji | jki.  Errors: SK_EINVAL.
 */
typedef enum { SK_PAIR_AUTO = 0, SK_PAIR_KJI = 1, SK_PAIR_JKI = 2 } sk_pair_path_t;
int sketch_set_pair_path(int path);

/* sketch_plan_host_jki -- as sketch_plan_host, but always builds the jki structure (for
 * measurements and tests of Algorithm 4 on any sparsity pattern).  Same errors, plus SK_EUNSUPPORTED
 * when the structure cannot be built (nnz >= 2^32 - 1, m > 2^27, more than 32767 column blocks). */
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
