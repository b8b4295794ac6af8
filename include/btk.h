/*
 * btk.h — C ABI of the B200-native bucketed approximate top-k library
 * (libbtk.so, built from paper_2412_04358_b200/csrc/).
 *
 * The reference (arxiv 2412.04358, /root/reference/pkg/src/bucketed_topk)
 * is a pure-Python/NumPy package with no native FFI; its plugin surface is
 * the Python API.  Each entry point below replaces one reference function
 * (file:line cited) with the same argument meaning and error codes; the
 * Python package paper_2412_04358_b200 binds them with ctypes (see
 * INTEGRATION.md for the binding a reference maintainer would add).
 *
 * Conventions
 *   - Plain pointers and sizes only.  All data pointers are DEVICE pointers
 *     (cudaMalloc / torch CUDA tensors); `stream` is a cudaStream_t passed as
 *     void* (NULL = legacy default stream).  Calls are asynchronous and
 *     stream-ordered; the library never allocates, never synchronises.
 *   - Scores: m rows of n elements, row r at x + r*row_stride elements,
 *     unit stride inside a row.  dtype: BTK_F32 / BTK_BF16 / BTK_F16 / BTK_F64.
 *   - Outputs are canonical: per row, value descending, ties by lower
 *     original index (reference exact.py:130-139); values are bit-exact
 *     copies of the selected inputs (sign of zero kept); indices int64.
 *   - Non-finite scores (NaN/+-inf; reference exact.py:94-95 raises
 *     NonFiniteInputError) set bit 0 of *nonfinite_flag (device uint32,
 *     may be NULL); results are then unspecified.  The caller reads the
 *     flag after the stream work completes.
 *   - Return value: BTK_OK or one of the error codes; codes 1..8 map 1:1 to
 *     the reference ConfigError.code strings (btk_error_code()).
 */
#ifndef BTK_H_
#define BTK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* BTK_F64: the reference's native dtype (exact.py:87-96 computes in
 * float64); exact, on a generic 128-bit-key path (btk_f64.cu). */
enum btk_dtype { BTK_F32 = 0, BTK_BF16 = 1, BTK_F16 = 2, BTK_F64 = 3 };

/* reference core.py:28-47 (Assignment) */
enum btk_layout { BTK_INTERLEAVED = 0, BTK_CONTIGUOUS = 1 };

enum btk_status {
  BTK_OK = 0,
  BTK_ERR_NONPOSITIVE = 1,             /* "nonpositive"   core.py:98-102 */
  BTK_ERR_K_GT_N = 2,                  /* "k_gt_n"        core.py:103-104 */
  BTK_ERR_B_GT_N = 3,                  /* "b_gt_n"        core.py:105-106 */
  BTK_ERR_KB_RANGE = 4,                /* "kb_range"      core.py:107-112 */
  BTK_ERR_UNDERSAMPLED = 5,            /* "undersampled"  core.py:113-116 */
  BTK_ERR_INSUFFICIENT_CANDIDATES = 6, /* approx.py:266-271 */
  BTK_ERR_CHUNKS_RANGE = 7,            /* approx.py:69-77 */
  BTK_ERR_ASSIGNMENT = 8,              /* core.py:39-47 */
  BTK_ERR_DTYPE = 9,                   /* unsupported dtype */
  BTK_ERR_SHAPE = 10,                  /* ValueError: shape (exact.py:92-93) */
  BTK_ERR_WORKSPACE = 11,              /* workspace too small / misaligned */
  BTK_ERR_ALIGNMENT = 12,              /* misaligned device pointer */
  BTK_ERR_CUDA = 13,                   /* CUDA launch error (see btk_last_cuda_error) */
  BTK_ERR_LABEL_RANGE = 14             /* carried label outside [0, 2^31-1] */
};

/* Joint validity of (m, n, k, b, k_b).  reference core.py:84-116
 * (check_parameters), same checks in the same order. */
int btk_validate(int64_t m, int64_t n, int64_t k, int64_t b, int64_t kb);

/* Stage-1-only validity (no k).  reference approx.py:216-224. */
int btk_stage1_validate(int64_t n, int64_t b, int64_t kb);

/* Stage-1 candidates per row: sum_j min(k_b, size_j).
 * reference core.py:155-158 (stage1_candidate_count). */
int64_t btk_stage1_count(int64_t n, int64_t b, int64_t kb, int layout);

/* Bytes of device workspace btk_approx_topk needs for ANY input pointer
 * and row stride of this shape (the worst case; 0 is possible — the fused
 * kernels need none).  Contents need not be initialised. */
size_t btk_workspace_bytes(int64_t m, int64_t n, int64_t k, int64_t b, int64_t kb, int dtype,
                           int layout);

/* Bytes of workspace the plan for exactly this call (input pointer
 * alignment and row stride included) needs: <= btk_workspace_bytes. */
size_t btk_plan_workspace_bytes(const void* x, int64_t row_stride, int dtype, int64_t m, int64_t n,
                                int64_t k, int64_t b, int64_t kb, int layout);

/* Bucketed approximate top-k: Stage 1 (per-bucket top-k_b) + Stage 2 (exact
 * top-k over the survivors, canonical order).
 * reference approx.py:245-282 (approx_topk).  out_vals: m x k (dtype),
 * out_idx: m x k int64, both row-contiguous. */
int btk_approx_topk(const void* x, int64_t row_stride, int dtype, int64_t m, int64_t n, int64_t k,
                    int64_t b, int64_t kb, int layout, void* out_vals, int64_t* out_idx, void* ws,
                    size_t ws_bytes, uint32_t* nonfinite_flag, void* stream);

/* Stage 1 only: (m, C) candidates in bucket-id order, each bucket's
 * min(k_b, size_j) survivors canonical.  reference approx.py:208-242
 * (stage1 / Stage1Candidates); C = btk_stage1_count(). */
size_t btk_stage1_workspace_bytes(int64_t m, int64_t n, int64_t b, int64_t kb, int dtype,
                                  int layout);
int btk_stage1(const void* x, int64_t row_stride, int dtype, int64_t m, int64_t n, int64_t b,
               int64_t kb, int layout, void* out_vals, int64_t* out_idx, void* ws,
               size_t ws_bytes, uint32_t* nonfinite_flag, void* stream);

/* btk_approx_topk with launch flags.  BTK_INPUT_READY: the caller
 * guarantees that `x` was not written by the work queued before this call
 * on `stream` (e.g. independent batches resident in HBM).  The kernels then
 * stream the input while the preceding kernel drains (programmatic
 * dependent launch) and wait for it only before their first global write,
 * so back-to-back launches overlap.  Results are identical either way. */
enum btk_launch_flags { BTK_INPUT_READY = 1 };
int btk_approx_topk_flags(const void* x, int64_t row_stride, int dtype, int64_t m, int64_t n,
                          int64_t k, int64_t b, int64_t kb, int layout, void* out_vals,
                          int64_t* out_idx, void* ws, size_t ws_bytes, uint32_t* nonfinite_flag,
                          uint32_t flags, void* stream);

/* Exact canonical top-k per row.  reference exact.py:162-173
 * (exact_topk_oracle); equals btk_approx_topk with b = 1, k_b = k. */
size_t btk_exact_workspace_bytes(int64_t m, int64_t n, int64_t k, int dtype);
int btk_exact_topk(const void* x, int64_t row_stride, int dtype, int64_t m, int64_t n, int64_t k,
                   void* out_vals, int64_t* out_idx, void* ws, size_t ws_bytes,
                   uint32_t* nonfinite_flag, void* stream);

/* Canonical top-k of (value, carried label) pairs.  reference
 * exact.py:142-159 (topk_with_indices).  Labels must lie in
 * [0, 2^31-1]; a label outside sets bit 1 of *flag. */
size_t btk_topk_with_indices_workspace_bytes(int64_t m, int64_t c, int64_t k, int dtype);
int btk_topk_with_indices(const void* values, const int64_t* labels, int dtype, int64_t m,
                          int64_t c, int64_t k, void* out_vals, int64_t* out_idx, void* ws,
                          size_t ws_bytes, uint32_t* flag, void* stream);

/* Recall counts of index rows (reference recall.py:203-218,
 * empirical_recall_rows): hits[r] = number of the k entries of approx row r
 * that occur among the k entries of truth row r (int64 indices, device
 * memory; row r at approx_idx + r*approx_stride).  No workspace. */
int btk_recall_hits(const int64_t* approx_idx, int64_t approx_stride, const int64_t* truth_idx,
                    int64_t truth_stride, int64_t m, int64_t k, int32_t* hits, void* stream);

/* Paper's total-bandwidth numerator (reference bench.py:138-159):
 * m * (n*vb + k*(vb + ib)). */
int64_t btk_min_bytes(int64_t m, int64_t n, int64_t k, int64_t value_bytes, int64_t index_bytes);

/* Which kernel family btk_approx_topk would run: 1 fused, 0 generic. */
int btk_uses_fused_path(int64_t m, int64_t n, int64_t k, int64_t b, int64_t kb, int dtype,
                        int layout, int64_t row_stride);

/* Which kernel family btk_approx_topk runs for this problem (diagnostic;
 * the tests assert every family is exercised).  -1 if invalid. */
enum btk_family {
  BTK_FAM_GENERIC = 0,     /* s1_generic (thread per bucket) + K2 */
  BTK_FAM_NARROW = 1,      /* fused_narrow: TMA ring, cluster of S CTAs per row */
  BTK_FAM_WIDE = 2,        /* fused_wide: one CTA per row, LDG vector columns */
  BTK_FAM_ROWS = 3,        /* fused_rows: one warp per row */
  BTK_FAM_VEC_POOL = 4,    /* s1_vec pool + K2 */
  BTK_FAM_MATERIALIZE = 5, /* b == 1 or k_b > 16: exact radix select per bucket straight from the
                              scores (nothing materialised; name kept for ABI stability) + K2 */
  BTK_FAM_F64 = 6,         /* float64: 128-bit keys (btk_f64.cu) */
  BTK_FAM_POOL_CHUNKED = 7, /* s1_vec pool + histogram-chunked Stage 2 (btk_pool.cu) */
  BTK_FAM_XCHG = 8,         /* value-range exchange (btk_xchg.cu): batched split / partition / owner-sort
                               launches (16-bit default), or fused_xchg, a DSMEM cluster per row */
  BTK_FAM_CONTIG = 9        /* s1_contig (contiguous layout, warp per bucket, 128-bit loads) + K2 */
};
int btk_kernel_family(int64_t m, int64_t n, int64_t k, int64_t b, int64_t kb, int dtype,
                      int layout, int64_t row_stride);

/* Number of kernel launches one btk_approx_topk call issues for this
 * problem (the bench's gpu_launches claim is derived from it). */
int btk_launch_count(int64_t m, int64_t n, int64_t k, int64_t b, int64_t kb, int dtype,
                     int layout, int64_t row_stride);

/* Error helpers: stable reference code string ("kb_range", ...) and a
 * human-readable message. */
const char* btk_error_code(int status);
const char* btk_error_string(int status);
int btk_last_cuda_error(void);

/* Library version / build tag. */
const char* btk_version(void);

#ifdef __cplusplus
}
#endif

#endif /* BTK_H_ */
