// CTA-level "Stage 2 + canonical order" engine: adaptive MSD bucketing of
// composite keys followed by in-bucket rank counting.
//
// Restates reference exact.py:130-159 (stable argsort by index, then
// stable argsort by -value, take k).  Composite keys (btk_common.cuh) are
// unique and their unsigned order IS that canonical order, so the job is
// "find the k largest keys of the pool, in descending order".
//
// Why not a radix sort: an LSD radix pass needs a stable per-digit rank
// (match.any + a serial smem counter chain per item), which profiled at
// ~70% of the large-k kernels.  Here, per range [lo, hi) of the pool:
//
//   1. keys -> registers; block min / max of the non-empty keys;
//   2. bucket d = (NB-1) - ((key - min) >> shift), with shift chosen so the
//      key range spans the NB buckets (range-adaptive: N(0,1) survivors or
//      tie-heavy rows spread evenly); smem atomics give each key a slot;
//   3. exclusive scan of the bucket counts -> every bucket's final position
//      range (the range already sits at its final global position);
//   4. scatter keys into bucket order (in place, from registers);
//   5. a key in a small bucket (<= RS_LIMIT) finds its final position as
//      bucket start + #{bucket keys greater than it} — lanes of a warp walk
//      the same bucket, so the smem reads are broadcasts;
//      larger buckets are queued and refined by the same procedure (each
//      level narrows the key range by >= 2^(lognb-1), so depth <= 6).
//
// Buckets that start at or beyond k are never ranked (selection for free).
// Empty slots (key 0) get a private last bucket and are never ranked.
// Result: inv[q] = pool position of the q-th largest key, q < min(k, #keys);
// RS_NONE beyond (read through rs_key -> 0, the empty key).  P <= 16384.
#pragma once

#include <cuda_fp16.h>

#include "btk_common.cuh"

namespace btk {

constexpr int RS_LIMIT = 64;    // largest bucket ranked by counting
constexpr int RS_WORK = 256;    // worklist capacity (ranges > RS_LIMIT are disjoint: <= P/65)
constexpr uint16_t RS_NONE = 0xFFFF;  // inv[q] when fewer than q+1 keys are non-empty

__device__ __forceinline__ uint64_t rs_key(const uint64_t* pool, uint16_t pos) {
  return pos == RS_NONE ? 0ull : pool[pos];
}

// #keys of bucket [s0, s1) ranked before key x at position p.  UNIQ: keys
// are unique (every composite key carries its index; only carried labels
// of topk_with_indices can repeat), so only "greater" counts.
template <bool UNIQ>
__device__ __forceinline__ int rs_count_greater(const uint64_t* pool, int s0, int s1, uint64_t x,
                                                int p) {
  int cnt = 0;
  if constexpr (UNIQ) {
#pragma unroll 4
    for (int j = s0; j < s1; ++j) cnt += pool[j] > x ? 1 : 0;
  } else {
    for (int j = s0; j < s1; ++j) {
      const uint64_t y = pool[j];
      cnt += (y > x || (y == x && j < p)) ? 1 : 0;
    }
  }
  return cnt;
}

struct RankSmem {
  uint64_t* pool;   // P keys (permuted in place)
  uint16_t* inv;    // >= k entries
  uint16_t* bid;    // P entries: bucket of each pool position (current level)
  uint32_t* hist;   // (1 << lognb) + 2 counters
  int2* work;       // RS_WORK ranges
  uint64_t* red;    // 3 * (NT / 32) words of scratch
  int* ctl;         // 2 ints: worklist head, tail
};

__device__ __forceinline__ int bits64(uint64_t v) { return v ? 64 - __clzll((long long)v) : 0; }

// Block-wide min / max of the non-empty keys and of their float values.
template <int NT>
__device__ __forceinline__ void block_minmax(uint64_t& mn, uint64_t& mx, float& vmn, float& vmx,
                                             uint64_t* red) {
  constexpr int NW = NT / 32;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint64_t a = __shfl_xor_sync(0xFFFFFFFFu, mn, o);
    const uint64_t b = __shfl_xor_sync(0xFFFFFFFFu, mx, o);
    const float c = __shfl_xor_sync(0xFFFFFFFFu, vmn, o);
    const float d = __shfl_xor_sync(0xFFFFFFFFu, vmx, o);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
    vmn = fminf(vmn, c);
    vmx = fmaxf(vmx, d);
  }
  const int w = threadIdx.x >> 5;
  float* fr = reinterpret_cast<float*>(red + 2 * NW);
  if ((threadIdx.x & 31) == 0) { red[w] = mn; red[NW + w] = mx; fr[w] = vmn; fr[NW + w] = vmx; }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    mn = red[i] < mn ? red[i] : mn;
    mx = red[NW + i] > mx ? red[NW + i] : mx;
    vmn = fminf(vmn, fr[i]);
    vmx = fmaxf(vmx, fr[NW + i]);
  }
  __syncthreads();
}

// Float value of a composite key (sign of zero dropped; only used to bucket).
template <int DT>
__device__ __forceinline__ float comp_value(uint64_t c, int ib) {
  const uint32_t bits = bits_of_key<DT>((uint32_t)(c >> (ib + 1)), 0u);
  if constexpr (DT == F32) return __uint_as_float(bits);
  else if constexpr (DT == BF16) return __uint_as_float(bits << 16);
  else return __half2float(__ushort_as_half((unsigned short)bits));
}

// In-place exclusive scan of a[0..len) by the whole CTA.
template <int NT>
__device__ __forceinline__ void block_exscan(uint32_t* a, int len, uint32_t* wsum) {
  constexpr int NW = NT / 32;
  const int chunk = (len + NT - 1) / NT;
  const int b0 = threadIdx.x * chunk;
  uint32_t s = 0;
  for (int i = 0; i < chunk; ++i) s += (b0 + i < len) ? a[b0 + i] : 0u;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  uint32_t wbase = 0;
#pragma unroll
  for (int i = 0; i < NW; ++i) wbase += (i < w) ? wsum[i] : 0u;
  uint32_t run = wbase + incl - s;
  for (int i = 0; i < chunk; ++i) {
    if (b0 + i < len) {
      const uint32_t c = a[b0 + i];
      a[b0 + i] = run;
      run += c;
    }
  }
  __syncthreads();
}

// Bucketing rule of one range.  Value mode (the default): buckets are
// uniform in the float VALUE between the range's min and max — IEEE
// subtraction / multiplication / floor are monotone, so bucket order never
// contradicts key order, equal values share a bucket, and typical score
// distributions spread evenly (key space is log-like in the value: a range
// crossing zero would waste most buckets on tiny magnitudes).  Key mode
// (all values equal, or a non-finite spread): uniform in key space, which
// then splits by index bits.
struct RsRule {
  uint64_t mn;
  float vmx, scale;
  int shift, nb;
  bool vmode, same;
};

template <int DT>
__device__ __forceinline__ int rs_bucket(const RsRule& r, uint64_t key, int ib) {
  if (!key) return r.nb;  // empty slots: private last bucket
  if (r.vmode) {
    const float t = (r.vmx - comp_value<DT>(key, ib)) * r.scale;
    return t < (float)(r.nb - 1) ? (int)t : r.nb - 1;
  }
  return (r.nb - 1) - (int)((key - r.mn) >> r.shift);
}

// Bucket one range [lo, hi) of the pool, rank its small buckets, queue the
// big ones.  All NT threads call it with identical arguments.
template <int DT, int NT, int ITEMS, bool UNIQ = true>
__device__ __forceinline__ void rs_range(const RankSmem& S, int lo, int hi, int k, int lognb,
                                         int ib) {
  const int tid = threadIdx.x;
  const int n = hi - lo;
  uint64_t key[ITEMS];
  uint32_t slot[ITEMS];
  uint64_t mn = ~0ull, mx = 0ull;
  float vmn = __int_as_float(0x7F800000), vmx = -__int_as_float(0x7F800000);
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int p = tid + i * NT;
    key[i] = (p < n) ? S.pool[lo + p] : 0ull;
    if (key[i]) {
      mn = key[i] < mn ? key[i] : mn;
      mx = key[i] > mx ? key[i] : mx;
      const float v = comp_value<DT>(key[i], ib);
      vmn = fminf(vmn, v);
      vmx = fmaxf(vmx, v);
    }
  }
  RsRule R;
  R.nb = 1 << lognb;
  for (int j = tid; j < R.nb + 2; j += NT) S.hist[j] = 0u;
  block_minmax<NT>(mn, mx, vmn, vmx, S.red);  // (its barriers also publish the clear)
  if (mx == 0ull) return;                     // nothing but empty slots
  R.mn = mn;
  R.vmx = vmx;
  R.same = (mn == mx);
  R.shift = max(0, bits64(mx - mn) - lognb);
  const float span = vmx - vmn;
  R.scale = (float)R.nb / span;
  // key space is already near-linear in the value inside one sign and
  // within a factor 4 of magnitude: use the cheaper key-space rule there
  const bool narrow_band = (vmn > 0.f && vmx < 4.f * vmn) || (vmx < 0.f && vmn > 4.f * vmx);
  R.vmode = !narrow_band && (span > 0.f) && (R.scale > 0.f) && (R.scale < 3.0e38f) &&
            (span < 3.0e38f);
  uint16_t dd[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int p = tid + i * NT;
    if (p < n) {
      dd[i] = (uint16_t)rs_bucket<DT>(R, key[i], ib);
      slot[i] = atomicAdd(&S.hist[dd[i]], 1u);
    }
  }
  __syncthreads();
  block_exscan<NT>(S.hist, R.nb + 2, reinterpret_cast<uint32_t*>(S.red));
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int p = tid + i * NT;
    if (p < n) {
      const int q = lo + (int)S.hist[dd[i]] + (int)slot[i];
      S.pool[q] = key[i];
      S.bid[q] = dd[i];
    }
  }
  __syncthreads();
  // rank pass over positions in bucket order
  for (int p = tid; p < n; p += NT) {
    const uint64_t x = S.pool[lo + p];
    if (!x) continue;
    if (R.same) {  // identical keys (duplicate carried labels): any order
      if (lo + p < k) S.inv[lo + p] = (uint16_t)(lo + p);
      continue;
    }
    const int d = S.bid[lo + p];
    const int s0 = (int)S.hist[d], s1 = (int)S.hist[d + 1];
    if (lo + s0 >= k) continue;  // bucket lies wholly beyond the k-th key
    if (s1 - s0 > RS_LIMIT) {
      if (p == s0) {
        const int t = atomicAdd(&S.ctl[1], 1);
        S.work[t % RS_WORK] = make_int2(lo + s0, lo + s1);
      }
      continue;
    }
    const int cnt = rs_count_greater<UNIQ>(S.pool + lo, s0, s1, x, p);
    const int f = lo + s0 + cnt;
    if (f < k) S.inv[f] = (uint16_t)(lo + p);
  }
  __syncthreads();
}

// Full engine: after return (and a barrier), inv[0 .. min(k, #non-empty))
// holds pool positions in canonical order.  P <= NT * ITEMS, P <= 16384.
// ib = index bits of the composite keys (CompGeo::ib).
template <int DT, int NT, int ITEMS, bool UNIQ = true>
__device__ void rank_select_sort(const RankSmem& S, int P, int k, int lognb, int ib) {
  if (threadIdx.x == 0) { S.ctl[0] = 0; S.ctl[1] = 0; }
  for (int q = threadIdx.x; q < k; q += NT) S.inv[q] = RS_NONE;
  __syncthreads();
  rs_range<DT, NT, ITEMS, UNIQ>(S, 0, P, k, lognb, ib);
  for (;;) {
    const int head = S.ctl[0], tail = S.ctl[1];
    if (head >= tail) break;
    const int2 r = S.work[head % RS_WORK];
    __syncthreads();
    if (threadIdx.x == 0) S.ctl[0] = head + 1;
    rs_range<DT, NT, ITEMS, UNIQ>(S, r.x, r.y, k, lognb, ib);
  }
  __syncthreads();
}

// Warp-synchronous form of the engine for one warp's pool of P <= 32*ITEMS
// keys (fused_rows; big buckets of k2_cluster): one bucketing level, then
// in-bucket counting with no size limit.  inv[f] = pos_off + position.
template <int DT, int ITEMS, bool UNIQ = true>
__device__ __forceinline__ void warp_rank_sort(uint64_t* pool, int P, int k, uint16_t* inv,
                                               uint16_t* bid, uint32_t* hist, int lognb, int ib,
                                               int pos_off = 0) {
  const int lane = threadIdx.x & 31;
  for (int q = lane; q < k && q < P; q += 32) inv[q] = RS_NONE;  // only this pool's slots
  uint64_t key[ITEMS];
  uint32_t slot[ITEMS];
  uint64_t mn = ~0ull, mx = 0ull;
  float vmn = __int_as_float(0x7F800000), vmx = -__int_as_float(0x7F800000);
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int p = lane + 32 * i;
    key[i] = p < P ? pool[p] : 0ull;
    if (key[i]) {
      mn = key[i] < mn ? key[i] : mn;
      mx = key[i] > mx ? key[i] : mx;
      const float v = comp_value<DT>(key[i], ib);
      vmn = fminf(vmn, v);
      vmx = fmaxf(vmx, v);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint64_t a = __shfl_xor_sync(0xFFFFFFFFu, mn, o);
    const uint64_t b = __shfl_xor_sync(0xFFFFFFFFu, mx, o);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
    vmn = fminf(vmn, __shfl_xor_sync(0xFFFFFFFFu, vmn, o));
    vmx = fmaxf(vmx, __shfl_xor_sync(0xFFFFFFFFu, vmx, o));
  }
  if (mx == 0ull) { __syncwarp(); return; }
  RsRule R;
  R.nb = 1 << lognb;
  R.mn = mn;
  R.vmx = vmx;
  R.same = (mn == mx);
  R.shift = max(0, bits64(mx - mn) - lognb);
  const float span = vmx - vmn;
  R.scale = (float)R.nb / span;
  const bool narrow_band = (vmn > 0.f && vmx < 4.f * vmn) || (vmx < 0.f && vmn > 4.f * vmx);
  R.vmode = !narrow_band && (span > 0.f) && (R.scale > 0.f) && (R.scale < 3.0e38f) &&
            (span < 3.0e38f);
  for (int j = lane; j < R.nb + 2; j += 32) hist[j] = 0u;
  __syncwarp();
  uint16_t dd[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (lane + 32 * i < P) {
      dd[i] = (uint16_t)rs_bucket<DT>(R, key[i], ib);
      slot[i] = atomicAdd(&hist[dd[i]], 1u);
    }
  }
  __syncwarp();
  {  // warp exclusive scan of hist[0 .. nb+2)
    const int len = R.nb + 2, chunk = (len + 31) / 32, b0 = lane * chunk;
    uint32_t sum = 0;
    for (int i = 0; i < chunk; ++i) sum += (b0 + i < len) ? hist[b0 + i] : 0u;
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += t;
    }
    uint32_t run = incl - sum;
    __syncwarp();
    for (int i = 0; i < chunk; ++i) {
      if (b0 + i < len) {
        const uint32_t c = hist[b0 + i];
        hist[b0 + i] = run;
        run += c;
      }
    }
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (lane + 32 * i < P) {
      const int q = (int)hist[dd[i]] + (int)slot[i];
      pool[q] = key[i];
      bid[q] = dd[i];
    }
  }
  __syncwarp();
  for (int p = lane; p < P; p += 32) {
    const uint64_t x = pool[p];
    if (!x) continue;
    if (R.same) {
      if (p < k) inv[p] = (uint16_t)(pos_off + p);
      continue;
    }
    const int d = bid[p];
    const int s0 = (int)hist[d], s1 = (int)hist[d + 1];
    if (s0 >= k) continue;
    const int cnt = rs_count_greater<UNIQ>(pool, s0, s1, x, p);
    const int f = s0 + cnt;
    if (f < k) inv[f] = (uint16_t)(pos_off + p);
  }
  __syncwarp();
}

// Shared-memory bytes the engine needs besides the pool (P keys).
__host__ __device__ constexpr size_t rank_aux_bytes(int nt, int lognb, int64_t k, int64_t P) {
  return ((size_t)((1 << lognb) + 2) * 4 + 127) / 128 * 128 +  // hist
         ((size_t)k * 2 + 127) / 128 * 128 +                   // inv
         ((size_t)P * 2 + 127) / 128 * 128 +                   // bid
         (size_t)RS_WORK * 8 + (size_t)(nt / 32) * 24 + 128;  // work, red, ctl
}

// Carve the engine's scratch out of `aux` (rank_aux_bytes of it).
__device__ __forceinline__ RankSmem rank_smem(uint64_t* pool, uint8_t* aux, int64_t P, int64_t k,
                                              int lognb, int nt) {
  RankSmem S;
  S.pool = pool;
  S.hist = reinterpret_cast<uint32_t*>(aux);
  aux += ((size_t)((1 << lognb) + 2) * 4 + 127) / 128 * 128;
  S.inv = reinterpret_cast<uint16_t*>(aux);
  aux += ((size_t)k * 2 + 127) / 128 * 128;
  S.bid = reinterpret_cast<uint16_t*>(aux);
  aux += ((size_t)P * 2 + 127) / 128 * 128;
  S.work = reinterpret_cast<int2*>(aux);
  aux += (size_t)RS_WORK * 8;
  S.red = reinterpret_cast<uint64_t*>(aux);
  aux += (size_t)(nt / 32) * 24;
  S.ctl = reinterpret_cast<int*>(aux);
  return S;
}

// Choose log2(#buckets) for a pool of P keys: ~2 keys per bucket, 256..4096
// (bucket ids are 16-bit; the in-bucket count costs ~bucket size per key).
__host__ __device__ inline int rank_lognb(int64_t P) {
  int l = 8;
  while (l < 12 && ((int64_t)1 << (l + 1)) < P) ++l;
  return l;
}

}  // namespace btk
