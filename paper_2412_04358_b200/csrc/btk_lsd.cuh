// CTA-level stable LSD radix machinery with per-thread shared-memory digit
// counters (no atomics, no match.any), shared by the cluster-exchange
// kernel's owner sort (btk_xchg.cu) and the wide kernel's large pools.
//
// Counters: cnt[q * NT + tid] packs the thread's counts of digits 2q (low
// 16 bits) and 2q+1 (high 16 bits), q < WORDS (2*WORDS digits).  Items are
// thread-BLOCKED (thread t owns consecutive positions), so ranking in
// (thread, item) order is the stable order.
//
// Descending composite-key sorts (reference exact.py:130-159: the two
// stable argsorts are "sort comps descending") can skip the low bits of
// the index field when the input is already ordered by them: for
// interleaved buckets idx = t*b + j with b a power of two, and a pool laid
// out in bucket-id order is sorted by ~j, so only bits >= 1 + log2(b) are
// passed over.
#pragma once

#include "btk_common.cuh"

namespace btk {
namespace lsd {

// Block-wide digit scan: on return cnt holds the thread's exclusive base per
// digit (within the digit, in thread order), tot[d] the block total of digit
// d, dex[d] the digit-concatenated exclusive base.  ws: NT/32 x WORDS.
template <int NT, int WORDS>
__device__ __forceinline__ void digit_scan(uint32_t* cnt, uint32_t (*ws)[WORDS], uint32_t* tot, uint32_t* dex) {
  constexpr int NW = NT / 32;
  static_assert(NW <= 32 && WORDS <= 32, "shape");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t own[WORDS], w[WORDS];
#pragma unroll
  for (int q = 0; q < WORDS; ++q) w[q] = own[q] = cnt[q * NT + tid];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
    for (int q = 0; q < WORDS; ++q) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, w[q], o);
      if (lane >= o) w[q] += t;
    }
  }
  if (lane == 31) {
#pragma unroll
    for (int q = 0; q < WORDS; ++q) ws[warp][q] = w[q];
  }
  __syncthreads();
  if (warp == 0) {  // lane q < WORDS: exclusive over warps of word q, then over digits
    uint32_t all = 0;
    if (lane < WORDS) {
      for (int ww = 0; ww < NW; ++ww) {
        const uint32_t v = ws[ww][lane];
        ws[ww][lane] = all;
        all += v;
      }
    }
    const uint32_t lo = all & 0xFFFFu, hi = all >> 16, pair = lo + hi;
    uint32_t e = pair;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, e, o);
      if (lane >= o) e += u;
    }
    e -= pair;
    if (lane < WORDS) {
      tot[2 * lane] = lo;
      tot[2 * lane + 1] = hi;
      dex[2 * lane] = e;
      dex[2 * lane + 1] = e + lo;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < WORDS; ++q) cnt[q * NT + tid] = w[q] - own[q] + ws[warp][q];
}

// digit_scan whose per-thread bases start at off[d] instead of 0 (a
// running offset per digit across rounds; bases stay below 2^16)
template <int NT, int WORDS>
__device__ __forceinline__ void digit_scan_from(uint32_t* cnt, uint32_t (*ws)[WORDS], uint32_t* tot, uint32_t* dex,
                                                const uint32_t* off) {
  digit_scan<NT, WORDS>(cnt, ws, tot, dex);
  const int tid = threadIdx.x;
#pragma unroll
  for (int q = 0; q < WORDS; ++q) cnt[q * NT + tid] += off[2 * q] | (off[2 * q + 1] << 16);
}

// count one item of digit d in the thread's counters; returns the number of
// the thread's earlier items with that digit
template <int NT>
__device__ __forceinline__ uint32_t count_digit(uint32_t* cnt, uint32_t d) {
  uint32_t* c = cnt + (d >> 1) * NT + threadIdx.x;
  const uint32_t sh = (d & 1u) << 4;
  const uint32_t v = *c;
  *c = v + (1u << sh);
  return (v >> sh) & 0xFFFFu;
}
template <int NT>
__device__ __forceinline__ uint32_t digit_base(const uint32_t* cnt, uint32_t d) {
  return (cnt[(d >> 1) * NT + threadIdx.x] >> ((d & 1u) << 4)) & 0xFFFFu;
}

// padded position: one slot of padding per 32, so thread-blocked runs of
// 32 u64 keys are (nearly) bank-conflict free
__host__ __device__ __forceinline__ int pad32(int p) { return p + (p >> 5); }

// In-place stable descending LSD sort of the N keys at keys[pad32(p)],
// p < N <= NT*ITEMS, over the bits >= lowbit that vary; RB-bit digits.
// Smem: cnt (WORDS*NT u32, WORDS = 2^(RB-1)), ws (NT/32 x WORDS), tot/dex
// (2*WORDS each), s_vary (one u64).  Positions >= N are treated as key 0.
template <int NT, int ITEMS, int RB>
__device__ __forceinline__ void sort_desc_inplace(uint64_t* keys, int N, int lowbit, uint32_t* cnt,
                                                  uint32_t (*ws)[1 << (RB - 1)], uint32_t* tot,
                                                  uint32_t* dex, unsigned long long* s_vary) {
  constexpr int DIG = 1 << RB, WORDS = DIG / 2;
  const int tid = threadIdx.x, lane = tid & 31;
  const int items = (N + NT - 1) / NT;
  uint64_t key[ITEMS];
  uint64_t vary = 0;
  if (tid == 0) *s_vary = 0ull;
  __syncthreads();
  const uint64_t k0 = N ? keys[0] : 0ull;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int p = tid * items + i;
    key[i] = (i < items && p < N) ? keys[pad32(p)] : 0ull;
    if (i < items && p < N) vary |= key[i] ^ k0;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) vary |= __shfl_xor_sync(0xFFFFFFFFu, vary, o);
  if (lane == 0 && vary) atomicOr(s_vary, (unsigned long long)vary);
  __syncthreads();
  vary = *s_vary;
  int shift = lowbit;
  if ((vary >> lowbit) != 0ull) shift = lowbit + __ffsll((long long)(vary >> lowbit)) - 1;
  for (; shift < 64 && (vary >> shift) != 0ull; shift += RB) {
    if (((vary >> shift) & (uint64_t)(DIG - 1)) == 0ull) continue;
    uint32_t dl[ITEMS];
#pragma unroll
    for (int q = 0; q < WORDS; ++q) cnt[q * NT + tid] = 0u;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      if (i < items) {
        const uint32_t d = (uint32_t)(DIG - 1) - (uint32_t)((key[i] >> shift) & (uint64_t)(DIG - 1));
        dl[i] = (d << 16) | count_digit<NT>(cnt, d);
      }
    }
    digit_scan<NT, WORDS>(cnt, ws, tot, dex);  // contains the barrier after every thread's reads
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      if (i < items) {
        const uint32_t d = dl[i] >> 16;
        const int r = (int)(dex[d] + digit_base<NT>(cnt, d) + (dl[i] & 0xFFFFu));
        if (r < N) keys[pad32(r)] = key[i];  // pads (key 0, last) beyond N are dropped
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int p = tid * items + i;
      key[i] = (i < items && p < N) ? keys[pad32(p)] : 0ull;
    }
  }
}

}  // namespace lsd
}  // namespace btk
