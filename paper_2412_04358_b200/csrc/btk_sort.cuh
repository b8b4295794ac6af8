// CTA-level LSD radix machinery over 64-bit composite keys (descending).
//
// This is the exact "Stage 2 + canonical order" engine (reference
// exact.py:130-159: stable argsort by index then stable argsort by -value,
// which for unique composite keys is just "sort comps descending").
//
// Layout: a tile of NT*ITEMS keys, warp w / lane l / item i holds logical
// position w*32*ITEMS + i*32 + l ("warp-striped": coalesced loads and a
// rank order that equals memory order, so every pass is stable).
// Ranking uses match.any per item with a warp-private 256-bin histogram:
// no atomics, deterministic.
#pragma once

#include "btk_common.cuh"

namespace btk {

constexpr int RADIX = 256;

// Digit of a key for a descending sort: rank ascending on ~key.
__device__ __forceinline__ uint32_t desc_digit(uint64_t key, int shift) {
  return (uint32_t)((~key) >> shift) & 0xFFu;
}

// Rank the ITEMS keys a thread holds within its warp.  whist_w is this warp's
// 256-counter row (cleared by the caller).  rank[i] = #keys before it in the
// warp's logical order with the same digit.  On return whist_w[d] holds the
// warp's count of digit d.
template <int ITEMS>
__device__ __forceinline__ void warp_rank(const uint64_t (&key)[ITEMS], int shift,
                                          uint32_t* whist_w, uint32_t (&rank)[ITEMS]) {
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    uint32_t d = desc_digit(key[i], shift);
    uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
    uint32_t before = __popc(peers & lt);
    uint32_t cnt = whist_w[d];
    rank[i] = cnt + before;
    __syncwarp();
    if (before == 0) whist_w[d] = cnt + __popc(peers);
    __syncwarp();
  }
}

// After all warps ranked: convert whist (NW x 256, counts) into per-warp
// exclusive offsets within each digit (digit-major, warp-minor) and fill
// dtotal[d] with the tile total of digit d.  Needs NT >= 256.
template <int NT>
__device__ __forceinline__ void warp_offsets(uint32_t* whist, uint32_t* dtotal) {
  constexpr int NW = NT / 32;
  for (int d = threadIdx.x; d < RADIX; d += NT) {
    uint32_t run = 0;
#pragma unroll 4
    for (int w = 0; w < NW; ++w) {
      uint32_t c = whist[w * RADIX + d];
      whist[w * RADIX + d] = run;
      run += c;
    }
    dtotal[d] = run;
  }
}

// Exclusive scan of 256 counters in place by one warp; returns (to lane 0
// caller via smem) nothing.  in/out may alias.
__device__ __forceinline__ void warp_exscan256(const uint32_t* in, uint32_t* out) {
  const int lane = threadIdx.x & 31;
  uint32_t v[8];
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) { v[j] = in[lane * 8 + j]; s += v[j]; }
  uint32_t incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += t;
  }
  uint32_t run = incl - s;
#pragma unroll
  for (int j = 0; j < 8; ++j) { uint32_t c = v[j]; out[lane * 8 + j] = run; run += c; }
}

// Sort NT*ITEMS keys held in smem (skeys) descending over bits
// [begin_bit, end_bit).  smem scratch: whist (NW*256), dbase, dtotal (256).
template <int NT, int ITEMS>
__device__ void block_sort_desc(uint64_t* skeys, uint32_t* whist, uint32_t* dbase,
                                uint32_t* dtotal, int begin_bit, int end_bit) {
  constexpr int N = NT * ITEMS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int base = warp * 32 * ITEMS + lane;
  uint64_t key[ITEMS];
  uint32_t rank[ITEMS];
  __shared__ int s_skip;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) key[i] = skeys[base + i * 32];
  for (int shift = begin_bit; shift < end_bit; shift += 8) {
    uint32_t* wh = whist + warp * RADIX;
#pragma unroll
    for (int j = lane; j < RADIX; j += 32) wh[j] = 0;
    __syncwarp();
    warp_rank<ITEMS>(key, shift, wh, rank);
    __syncthreads();
    warp_offsets<NT>(whist, dtotal);
    if (threadIdx.x == 0) s_skip = 0;
    __syncthreads();
    if (warp == 0) warp_exscan256(dtotal, dbase);
    if (threadIdx.x < RADIX && dtotal[threadIdx.x] == (uint32_t)N) s_skip = 1;
    __syncthreads();
    if (s_skip) continue;  // every key has the same digit: pass is the identity
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      uint32_t d = desc_digit(key[i], shift);
      skeys[dbase[d] + whist[warp * RADIX + d] + rank[i]] = key[i];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) key[i] = skeys[base + i * 32];
    __syncthreads();  // whist/dbase reused next pass
  }
}

// Warp-parallel search over a 256-bin histogram for the bin where the
// cumulative count from the TOP (bin 255 downwards) reaches `need`.
// Returns the bin in *out_bin and the count strictly above it in *out_above.
// Called by one full warp.
__device__ __forceinline__ void find_crossing_desc(const uint32_t* hist, uint32_t need,
                                                   int* out_bin, uint32_t* out_above) {
  const int lane = threadIdx.x & 31;
  // lane L covers bins [255 - 8L - 7, 255 - 8L] scanned top-down.
  uint32_t v[8];
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) { v[j] = hist[255 - lane * 8 - j]; s += v[j]; }
  uint32_t incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += t;
  }
  uint32_t excl = incl - s;
  bool mine = (excl < need) && (incl >= need);
  if (mine) {
    uint32_t run = excl;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (run + v[j] >= need) { *out_bin = 255 - lane * 8 - j; *out_above = run; break; }
      run += v[j];
    }
  }
}

}  // namespace btk
