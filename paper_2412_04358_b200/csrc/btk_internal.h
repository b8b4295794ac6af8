// Internal (non-ABI) declarations shared by the library's translation units.
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "btk_common.cuh"

namespace btk {

// Longest segment K2 sorts entirely in one CTA's shared memory.
constexpr int64_t K2_SMALL_CAP = 16384;

// Chunked Stage 2 for large pools (btk_pool.cu): coarse bins = the top
// POOL_HBITS bits of a composite key (8 bf16/fp16 values or 2^19 fp32
// ulps per bin); chunks of whole bins start at multiples of POOL_HALF
// selected keys, so a chunk holds < 2 * POOL_HALF keys when no selected
// bin exceeds POOL_HALF (else the row takes the radix-select fallback).
constexpr int POOL_HBITS = 13;
constexpr int POOL_HALF = 8192;
constexpr int POOL_MAXC = 16;  // chunks per row (k <= (POOL_MAXC - 1) * POOL_HALF)
struct ChunkTab {
  int n;                      // chunks (-1: this row takes the fallback)
  int start[POOL_MAXC + 1];   // output offset of chunk c (= its offset in the chunk buffer)
  int pad[2];
};

struct K2Args {
  const uint64_t* in;   // nseg segments of L keys (row stride in_stride)
  int64_t in_stride;
  int64_t nseg;
  int64_t L;
  int64_t kk;           // keep the kk largest, sorted descending
  uint64_t* out_keys;   // !decode: nseg x kk comps (row stride out_stride)
  void* out_vals;       // decode: values (input dtype) ...
  int64_t* out_idx;     //         ... and int64 indices
  int64_t out_stride;
  CompGeo geo;
  uint64_t* scratch_a;  // long segments only: nseg * kk keys each
  uint64_t* scratch_b;
  bool unique = true;   // keys unique (false: repeated carried labels possible)
  // optional row mask: segment s runs only if mask[s * mask_stride] < 0
  // (the chunked Stage 2's fallback rows); scratch_b may use its own stride
  const int* mask = nullptr;
  int64_t mask_stride = 0;
  int64_t scratch_a_stride = 0;  // 0: kk
  int64_t scratch_b_stride = 0;  // 0: kk
};

// Opt a kernel into >48 KB dynamic smem once per device (never during
// stream capture, where the warm-up call has already done it).
inline cudaError_t ensure_smem_attr(const void* fn, size_t bytes) {
  if (bytes == 0) return cudaSuccess;
  static thread_local const void* done_fn[64];
  static thread_local int done_dev[64];
  static thread_local int n_done = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  for (int i = 0; i < n_done; ++i)
    if (done_fn[i] == fn && done_dev[i] == dev) return cudaSuccess;
  // opt in to the full 227 KB once; the per-launch size still sets occupancy
  (void)bytes;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
  if (e == cudaSuccess && n_done < 64) { done_fn[n_done] = fn; done_dev[n_done] = dev; ++n_done; }
  return e;
}

cudaError_t run_k2(int dtype, bool decode, const K2Args& a, cudaStream_t st);
// Exact top-kk composite keys of each of the nb buckets of m raw score
// rows, unsorted (0 = empty), into out[m*nb][kk] — no materialisation of
// the rows' n keys; K2 then sorts them.  nb = 1: whole rows.
cudaError_t run_select_raw(int dtype, const void* x, int64_t row_stride, int64_t m, int64_t n, int64_t nb,
                           int layout, int64_t kk, uint64_t* out, CompGeo g, uint32_t* flag, cudaStream_t st);
cudaError_t run_decode(int dtype, const uint64_t* in, int64_t in_stride, int64_t nseg, int64_t kk,
                       void* out_vals, int64_t* out_idx, int64_t out_stride, CompGeo g,
                       cudaStream_t st);

// Problem description shared by the stage-1 launchers.
struct Problem {
  const void* x;
  int64_t row_stride;  // elements
  int dtype;
  int64_t m, n, k, b, kb;
  int layout;          // 0 interleaved, 1 contiguous
  CompGeo geo;
  uint32_t* flag;      // device non-finite flag (may be null)
  uint32_t flags = 0;  // BTK_INPUT_READY: input not produced by the preceding stream work
};

// Generic stage 1, k_b <= 16: one thread per (row, bucket), register queue.
// pool: m x (b*kb) comps, bucket-major, sorted within bucket, 0 = empty.
cudaError_t run_stage1_generic(const Problem& p, uint64_t* pool, cudaStream_t st);
// Contiguous layout, k_b <= 8: one warp per (row, bucket), 128-bit loads
// of the dense slice, warp merge of the lanes' queues.  Same pool layout.
bool stage1_contig_supported(const Problem& p);
cudaError_t run_stage1_contig(const Problem& p, uint64_t* pool, cudaStream_t st);
// Vectorised stage 1 into the same pool (interleaved, k_b in {1,2,4,8},
// V*k_b <= 16, 16-byte aligned rows); cudaErrorNotSupported otherwise.
bool stage1_vec_supported(const Problem& p);
cudaError_t run_stage1_vec(const Problem& p, uint64_t* pool, cudaStream_t st,
                           uint32_t* hist = nullptr, const int* rowmask = nullptr);
// Cluster-exchange fused kernel for large pools (btk_xchg.cu): Stage 1 and
// Stage 2 of a row in one cluster launch, plus the row-masked generic
// fallback for rows whose value partition overflows.
// kernel launches of one call on the exchange family: the batched pipeline
// (split, then partition + sort per batch of rows, fallback) or the cluster
// kernel + fallback
int xchg_launch_count(const Problem& p);
bool xchg_supported(const Problem& p);
size_t xchg_workspace_bytes(const Problem& p);
cudaError_t run_xchg(const Problem& p, void* ws, void* out_vals, int64_t* out_idx, cudaStream_t st);
// Chunked Stage 2 over a stage-1 pool with its coarse histogram.
bool pool_chunked_ok(const Problem& p);
size_t pool_chunked_bytes(const Problem& p);  // hist + tab + chunk buffer
cudaError_t run_pool_chunked(const Problem& p, uint64_t* pool, void* ws, void* out_vals,
                             int64_t* out_idx, cudaStream_t st);
// pool (m x b*kb) -> compact (m x C) values/indices in bucket order.
cudaError_t run_stage1_emit(const Problem& p, const uint64_t* pool, int64_t C, void* out_vals,
                            int64_t* out_idx, cudaStream_t st);
// Fused interleaved fast path (stage 1 + stage 2 in one kernel per row group).
// Returns cudaErrorNotSupported when the shape is outside its envelope.
// ws: fused_workspace_bytes(p) bytes, 256-aligned, zero-filled before first
// use (the split kernel's row counters; every call leaves them zero).
cudaError_t run_fused(const Problem& p, void* out_vals, int64_t* out_idx, void* ws, size_t ws_bytes,
                      cudaStream_t st);
bool fused_supported(const Problem& p);
// Fused kernel the planner picks: 0 none, 1 narrow, 2 wide, 3 rows.
int fused_kind(const Problem& p);
size_t fused_workspace_bytes(const Problem& p);

// Exact float64 path (btk_f64.cu): 128-bit composite keys.
size_t f64_workspace_bytes(int64_t m, int64_t n, int64_t k, int64_t b, int64_t kb);
size_t f64_stage1_workspace_bytes(int64_t m, int64_t n, int64_t b, int64_t kb);
size_t f64_pairs_workspace_bytes(int64_t m, int64_t c, int64_t k);
cudaError_t f64_approx_topk(const void* x, int64_t row_stride, int64_t m, int64_t n, int64_t k, int64_t b,
                            int64_t kb, int layout, void* out_vals, int64_t* out_idx, void* ws,
                            uint32_t* flag, cudaStream_t st);
cudaError_t f64_stage1(const void* x, int64_t row_stride, int64_t m, int64_t n, int64_t b, int64_t kb,
                       int layout, int64_t C, void* out_vals, int64_t* out_idx, void* ws, uint32_t* flag,
                       cudaStream_t st);
cudaError_t f64_topk_with_indices(const void* values, const int64_t* labels, int64_t m, int64_t c,
                                  int64_t k, void* out_vals, int64_t* out_idx, void* ws, uint32_t* flag,
                                  cudaStream_t st);

}  // namespace btk
