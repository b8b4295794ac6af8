// Per-row recall counts: |{a in approx row : a in truth row}| for index
// rows of length k (reference recall.py:203-218, empirical_recall_rows:
// for every approx index, is it among the truth indices — a searchsorted
// membership test, so a repeated approx index counts each time).
//
// One CTA per row.  The truth row is taken in chunks of CH indices, each
// chunk inserted into an open-addressing hash set in shared memory
// (atomicCAS on 64-bit keys, linear probing); every approx index of the
// current approx chunk (AC = 32 per thread, its "found" bits in one
// register) probes it.  Found bits accumulate across truth chunks, so a
// truth index repeated in two chunks is not counted twice.
#include "../../include/btk.h"
#include "btk_internal.h"

namespace btk {
namespace {

constexpr int RC_NT = 256;
constexpr int RC_AC = RC_NT * 32;  // approx indices per pass (one bit each per thread)
constexpr uint64_t EMPTY = ~0ull;

__device__ __forceinline__ uint32_t slot_of(uint64_t x, uint32_t mask) {
  return (uint32_t)((x * 0x9E3779B97F4A7C15ull) >> 32) & mask;
}

__global__ void __launch_bounds__(RC_NT) recall_hits(const int64_t* __restrict__ approx, int64_t astride,
                                                     const int64_t* __restrict__ truth, int64_t tstride,
                                                     int64_t k, int tb_log2, int32_t* __restrict__ hits) {
  extern __shared__ __align__(16) unsigned long long table[];
  __shared__ int s_has_empty;  // the truth chunk holds the sentinel value itself (index -1)
  __shared__ int s_sum;
  const int tid = threadIdx.x;
  const uint32_t TB = 1u << tb_log2, mask = TB - 1u;
  const int64_t CH = TB / 2;
  const int64_t* a = approx + blockIdx.x * astride;
  const int64_t* t = truth + blockIdx.x * tstride;
  if (tid == 0) s_sum = 0;
  int total = 0;
  for (int64_t a0 = 0; a0 < k; a0 += RC_AC) {
    uint32_t found = 0;
    for (int64_t t0 = 0; t0 < k; t0 += CH) {
      for (uint32_t i = tid; i < TB; i += RC_NT) table[i] = EMPTY;
      if (tid == 0) s_has_empty = 0;
      __syncthreads();
      const int64_t tn = min(CH, k - t0);
      for (int64_t i = tid; i < tn; i += RC_NT) {
        const uint64_t x = (uint64_t)t[t0 + i];
        if (x == EMPTY) { s_has_empty = 1; continue; }
        uint32_t s = slot_of(x, mask);
        while (true) {
          const unsigned long long prev = atomicCAS(&table[s], EMPTY, (unsigned long long)x);
          if (prev == EMPTY || prev == x) break;
          s = (s + 1u) & mask;
        }
      }
      __syncthreads();
#pragma unroll 4
      for (int q = 0; q < 32; ++q) {
        const int64_t e = a0 + (int64_t)q * RC_NT + tid;
        if (e >= k || ((found >> q) & 1u)) continue;
        const uint64_t x = (uint64_t)a[e];
        bool hit = false;
        if (x == EMPTY) {
          hit = s_has_empty != 0;
        } else {
          uint32_t s = slot_of(x, mask);
          while (true) {
            const uint64_t v = table[s];
            if (v == x) { hit = true; break; }
            if (v == EMPTY) break;
            s = (s + 1u) & mask;
          }
        }
        if (hit) found |= 1u << q;
      }
      __syncthreads();
    }
    total += __popc(found);
  }
  atomicAdd(&s_sum, total);
  __syncthreads();
  if (tid == 0) hits[blockIdx.x] = s_sum;
}

}  // namespace
}  // namespace btk

extern "C" int btk_recall_hits(const int64_t* approx_idx, int64_t approx_stride, const int64_t* truth_idx,
                               int64_t truth_stride, int64_t m, int64_t k, int32_t* hits, void* stream) {
  if (m < 1 || k < 1 || !approx_idx || !truth_idx || !hits) return BTK_ERR_SHAPE;
  if (approx_stride < k || truth_stride < k || m > 0x7FFFFFFF) return BTK_ERR_SHAPE;
  int lg = 1;  // table of 2 * min(k, 8192) slots, a power of two
  while ((int64_t(1) << lg) < 2 * std::min<int64_t>(k, 8192)) ++lg;
  const size_t smem = (size_t(1) << lg) * 8;
  const void* fn = (const void*)btk::recall_hits;
  if (btk::ensure_smem_attr(fn, smem) != cudaSuccess) return BTK_ERR_CUDA;
  btk::recall_hits<<<(unsigned)m, btk::RC_NT, smem, static_cast<cudaStream_t>(stream)>>>(
      approx_idx, approx_stride, truth_idx, truth_stride, k, lg, hits);
  return cudaGetLastError() == cudaSuccess ? BTK_OK : BTK_ERR_CUDA;
}
