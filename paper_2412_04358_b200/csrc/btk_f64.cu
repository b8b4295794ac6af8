// Exact float64 path (the reference's native dtype: exact.py:87-96 upcasts
// every input to float64, and its own callers — simdata._normal_rows,
// bench.time_selection, recall.monte_carlo_recall — pass float64).
//
// A float64 score cannot share the 64-bit composite key of the 32/16-bit
// paths (64 value bits alone), so this path orders 128-bit keys:
//
//   hi = vkey64(bits)                       order-preserving, -0 folded to +0
//   lo = (2^31-1 - label) << 33 | (2^32-1 - pos) << 1 | negzero
//
// label = original index (approx / exact paths, pos = 0) or the carried
// label (topk_with_indices, pos = position in the row, so repeated labels
// keep the stable-argsort order of exact.py:130-139).  Keys are unique and
// their unsigned order is the reference's total order; {0, 0} = empty.
//
// Kernels (all generic over layout, raggedness and row stride):
//   f64_s1_queue<KB>  Stage 1, k_b <= 16: one thread per (row, bucket),
//                     register insertion queue (reference approx.py:142-173).
//   f64_seg_small     segmented top-kk, segment <= 8192 keys: one CTA,
//                     keys in shared memory, bitonic sort descending.
//   f64_seg_select    longer segments: MSD radix select of the kk-th key
//                     (8-bit digits, shared histograms), compaction.
//   f64_lsd           kk > 8192: stable LSD radix sort through a global
//                     ping-pong buffer (exact.py:130-139's stable sorts).
// Segments are read straight from the scores (RowSrc: a bucket of a row,
// or the whole row when b == 1), so nothing is materialised.
#include <cstdint>

#include "../../include/btk.h"
#include "btk_internal.h"

namespace btk {
namespace f64 {

struct K128 {
  uint64_t hi, lo;
};

__device__ __forceinline__ bool kgt(const K128& a, const K128& b) {
  return a.hi > b.hi || (a.hi == b.hi && a.lo > b.lo);
}
__device__ __forceinline__ bool kempty(const K128& a) { return (a.hi | a.lo) == 0ull; }

constexpr uint64_t SIGN = 0x8000000000000000ull;
constexpr uint64_t EXPM = 0x7FF0000000000000ull;

__host__ __device__ __forceinline__ uint64_t vkey64(uint64_t bits) {
  bits = (bits == SIGN) ? 0ull : bits;
  return (bits & SIGN) ? ~bits : (bits | SIGN);
}

__device__ __forceinline__ K128 make_key(uint64_t bits, uint32_t label, uint32_t pos) {
  K128 k;
  k.hi = vkey64(bits);
  k.lo = ((uint64_t)(0x7FFFFFFFu - label) << 33) | ((uint64_t)(0xFFFFFFFFu - pos) << 1) |
         (bits == SIGN ? 1ull : 0ull);
  return k;
}

__device__ __forceinline__ void decode(const K128& k, uint64_t& bits, int64_t& label) {
  label = (int64_t)(0x7FFFFFFFu - (uint32_t)(k.lo >> 33));
  if (k.lo & 1ull) bits = SIGN;
  else bits = (k.hi & SIGN) ? (k.hi ^ SIGN) : ~k.hi;
}

// 8-bit digit of a 128-bit key at bit offset `shift` (multiple of 8).
__device__ __forceinline__ uint32_t digit(const K128& k, int shift) {
  return shift >= 64 ? (uint32_t)(k.hi >> (shift - 64)) & 0xFFu : (uint32_t)(k.lo >> shift) & 0xFFu;
}

// key >> shift as a 128-bit number (the MSD prefix), shift in [0, 128].
__device__ __forceinline__ K128 prefix_of(const K128& k, int shift) {
  K128 r;
  if (shift >= 128) { r.hi = r.lo = 0; return r; }
  if (shift >= 64) { r.lo = k.hi >> (shift - 64); r.hi = 0; return r; }  // value of key >> shift
  if (shift == 0) return k;
  r.lo = (k.lo >> shift) | (k.hi << (64 - shift));
  r.hi = k.hi >> shift;
  return r;
}

__device__ __forceinline__ bool keq(const K128& a, const K128& b) { return a.hi == b.hi && a.lo == b.lo; }

__device__ __forceinline__ bool nonfinite64(uint64_t bits) { return (bits & EXPM) == EXPM; }

// ------------------------------------------------------------------ sources
// One segment = one bucket of one row (or the whole row when b == 1).
struct RowSrc {
  const uint64_t* x;  // float64 bits
  int64_t row_stride, n, b;
  int layout;
  __device__ __forceinline__ void span(int64_t j, int64_t& start, int64_t& size, int64_t& step) const {
    if (layout == 0) {
      const int64_t q = n / b, r = n % b;
      start = j; size = q + (j < r ? 1 : 0); step = b;
    } else {
      start = (j * n + b - 1) / b;
      size = ((j + 1) * n + b - 1) / b - start;
      step = 1;
    }
  }
  struct Seg {
    const uint64_t* row;
    int64_t start, size, step;
    __device__ __forceinline__ int64_t len() const { return size; }
    __device__ __forceinline__ K128 get(int64_t p, bool& bad) const {
      const int64_t idx = start + p * step;
      const uint64_t bits = __ldg(reinterpret_cast<const unsigned long long*>(row) + idx);
      bad |= nonfinite64(bits);
      return make_key(bits, (uint32_t)idx, 0u);
    }
  };
  __device__ __forceinline__ Seg seg(int64_t s) const {
    Seg g;
    const int64_t row = s / b, j = s - row * b;
    g.row = x + row * row_stride;
    span(j, g.start, g.size, g.step);
    return g;
  }
};

// Keys already built (the Stage-1 pool, or compacted survivors).
struct KeySrc {
  const K128* k;
  int64_t stride, L;
  struct Seg {
    const K128* p;
    int64_t L;
    __device__ __forceinline__ int64_t len() const { return L; }
    __device__ __forceinline__ K128 get(int64_t q, bool&) const { return p[q]; }
  };
  __device__ __forceinline__ Seg seg(int64_t s) const { return Seg{k + s * stride, L}; }
};

// (value, carried label) pairs of topk_with_indices.
struct PairSrc {
  const uint64_t* v;
  const int64_t* lab;
  int64_t c;
  struct Seg {
    const uint64_t* v;
    const int64_t* lab;
    int64_t c;
    __device__ __forceinline__ int64_t len() const { return c; }
    __device__ __forceinline__ K128 get(int64_t p, bool& bad) const {
      const uint64_t bits = v[p];
      const int64_t l = lab[p];
      bad |= nonfinite64(bits);
      return make_key(bits, (uint32_t)(l < 0 ? 0 : (l > 0x7FFFFFFF ? 0x7FFFFFFF : l)), (uint32_t)p);
    }
  };
  __device__ __forceinline__ Seg seg(int64_t s) const { return Seg{v + s * c, lab + s * c, c}; }
};

// Output: either keys (kk per segment) or decoded (values, labels).
struct Out {
  K128* keys;          // non-null: write keys
  uint64_t* vals;      // else decoded
  int64_t* idx;
  int64_t stride;
  __device__ __forceinline__ void put(int64_t s, int64_t q, const K128& k) const {
    if (keys) {
      keys[s * stride + q] = k;
    } else {
      uint64_t bits;
      int64_t lab;
      if (kempty(k)) { bits = 0xFFF0000000000000ull; lab = -1; }  // never for validated shapes
      else decode(k, bits, lab);
      vals[s * stride + q] = bits;
      idx[s * stride + q] = lab;
    }
  }
};

constexpr int SMALL_CAP = 8192;  // keys sorted in one CTA's shared memory (128 KB)

__device__ __forceinline__ void flag_bad(bool bad, uint32_t* flag) {
  if (__syncthreads_or(bad) && threadIdx.x == 0 && flag) atomicOr(flag, 1u);
}

// ------------------------------------------------------------------ Stage 1, k_b <= 16
template <int KB>
__global__ void __launch_bounds__(256) f64_s1_queue(RowSrc src, int64_t m, int64_t kb, K128* pool,
                                                     uint32_t* flag) {
  const int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x;
  bool bad = false;
  for (int64_t row = blockIdx.y; row < m; row += gridDim.y) {
    if (j < src.b) {
      const RowSrc::Seg g = src.seg(row * src.b + j);
      K128 q[KB];
#pragma unroll
      for (int i = 0; i < KB; ++i) q[i] = K128{0ull, 0ull};
      for (int64_t t = 0; t < g.size; ++t) {
        const K128 c = g.get(t, bad);
        if (kgt(c, q[KB - 1])) {
#pragma unroll
          for (int i = KB - 1; i > 0; --i) q[i] = kgt(c, q[i - 1]) ? q[i - 1] : (kgt(c, q[i]) ? c : q[i]);
          q[0] = kgt(c, q[0]) ? c : q[0];
        }
      }
      K128* dst = pool + (row * src.b + j) * kb;
#pragma unroll
      for (int i = 0; i < KB; ++i)
        if (i < kb) dst[i] = q[i];
    }
  }
  flag_bad(bad, flag);
}

// ------------------------------------------------------------------ small segments
// Bitonic sort (descending) of P2 >= L keys in shared memory, keep kk.
template <int NT, class Src>
__global__ void __launch_bounds__(NT) f64_seg_small(Src src, int p2, int64_t kk, Out out, uint32_t* flag) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  K128* sk = reinterpret_cast<K128*>(smem_raw);
  const int64_t s = blockIdx.x;
  const auto g = src.seg(s);
  const int L = (int)g.len();
  bool bad = false;
  for (int p = threadIdx.x; p < p2; p += NT) sk[p] = (p < L) ? g.get(p, bad) : K128{0ull, 0ull};
  __syncthreads();
  for (int size = 2; size <= p2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < (p2 >> 1); t += NT) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool desc = ((lo & size) == 0);  // descending runs first
        const K128 a = sk[lo], b = sk[hi];
        const bool swap = desc ? kgt(b, a) : kgt(a, b);
        if (swap) { sk[lo] = b; sk[hi] = a; }
      }
      __syncthreads();
    }
  }
  for (int64_t q = threadIdx.x; q < kk; q += NT) out.put(s, q, q < p2 ? sk[q] : K128{0ull, 0ull});
  flag_bad(bad, flag);
}

// ------------------------------------------------------------------ long segments
// MSD radix select of the kk-th largest key, then compaction of the kk
// largest (unique keys; empty keys only as padding) to dst (kk per segment).
template <int NT, class Src>
__global__ void __launch_bounds__(NT) f64_seg_select(Src src, int64_t kk, K128* dst, uint32_t* flag) {
  __shared__ uint32_t hist[256];
  __shared__ uint32_t s_cnt;
  __shared__ int s_bin;
  __shared__ uint32_t s_above;
  const int64_t s = blockIdx.x;
  const auto g = src.seg(s);
  const int64_t L = g.len();
  K128* out = dst + s * kk;
  bool bad = false;
  if (L <= kk) {  // everything survives (ragged short buckets): copy + pad
    for (int64_t p = threadIdx.x; p < kk; p += NT) out[p] = (p < L) ? g.get(p, bad) : K128{0ull, 0ull};
    flag_bad(bad, flag);
    return;
  }
  K128 prefix{0ull, 0ull};
  uint32_t need = (uint32_t)kk;
  int shift = 128;
  bool early = false;
  while (shift > 0) {
    shift -= 8;
    for (int j = threadIdx.x; j < 256; j += NT) hist[j] = 0;
    __syncthreads();
    for (int64_t p = threadIdx.x; p < L; p += NT) {
      const K128 key = g.get(p, bad);
      if (keq(prefix_of(key, shift + 8), prefix)) atomicAdd(&hist[digit(key, shift)], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      // top-down crossing of `need`
      const int lane = threadIdx.x;
      uint32_t v[8], sum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) { v[q] = hist[255 - lane * 8 - q]; sum += v[q]; }
      uint32_t incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += t;
      }
      const uint32_t excl = incl - sum;
      if (excl < need && incl >= need) {
        uint32_t run = excl;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (run + v[q] >= need) { s_bin = 255 - lane * 8 - q; s_above = run; break; }
          run += v[q];
        }
      }
    }
    __syncthreads();
    const int bin = s_bin;
    need -= s_above;
    // prefix = (prefix << 8) | bin
    prefix.hi = (prefix.hi << 8) | (prefix.lo >> 56);
    prefix.lo = (prefix.lo << 8) | (uint64_t)bin;
    const uint32_t inbin = hist[bin];
    __syncthreads();
    if (inbin == need) { early = true; break; }
  }
  // selected: prefix_of(key, shift) > prefix, or == prefix (early: all of
  // the bin; else the threshold key itself, exact at shift 0)
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int64_t p0 = 0; p0 < L; p0 += NT) {
    const int64_t p = p0 + threadIdx.x;
    bool take = false;
    K128 key{0ull, 0ull};
    if (p < L) {
      key = g.get(p, bad);
      const K128 pk = prefix_of(key, shift);
      take = kgt(pk, prefix) || keq(pk, prefix);
      (void)early;
    }
    const uint32_t ball = __ballot_sync(0xFFFFFFFFu, take);
    uint32_t base = 0;
    if (lane == 0 && ball) base = atomicAdd(&s_cnt, (uint32_t)__popc(ball));
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    if (take) out[base + __popc(ball & lanemask_lt())] = key;
  }
  __syncthreads();
  for (int64_t p = s_cnt + threadIdx.x; p < kk; p += NT) out[p] = K128{0ull, 0ull};
  flag_bad(bad, flag);
}

// Stable LSD radix sort (descending) of kk keys per segment, ping-pong
// A <-> B, one CTA per segment, tiles of NT keys; the result is emitted.
template <int NT>
__global__ void __launch_bounds__(NT) f64_lsd(K128* A, K128* B, int64_t kk, Out out) {
  constexpr int NW = NT / 32;
  __shared__ uint32_t ghist[256];
  __shared__ uint32_t runbase[256];
  __shared__ uint32_t whist[NW][256];
  const int64_t s = blockIdx.x;
  K128* src = A + s * kk;
  K128* dst = B + s * kk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  for (int shift = 0; shift < 128; shift += 8) {
    for (int j = threadIdx.x; j < 256; j += NT) ghist[j] = 0;
    __syncthreads();
    for (int64_t p = threadIdx.x; p < kk; p += NT) atomicAdd(&ghist[255u - digit(src[p], shift)], 1u);
    __syncthreads();
    // block-uniform skip verdict (no shared flag: a reset by thread 0 at the
    // next pass would race with the readers of this one)
    const bool full = threadIdx.x < 256 && ghist[threadIdx.x] == (uint32_t)kk;
    if (warp == 0) {  // exclusive scan of ghist -> runbase
      uint32_t v[8], sum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) { v[q] = ghist[lane * 8 + q]; sum += v[q]; }
      uint32_t incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += t;
      }
      uint32_t run = incl - sum;
#pragma unroll
      for (int q = 0; q < 8; ++q) { runbase[lane * 8 + q] = run; run += v[q]; }
    }
    if (__syncthreads_or(full)) continue;
    for (int64_t t0 = 0; t0 < kk; t0 += NT) {
      const int64_t p = t0 + threadIdx.x;
      const bool valid = p < kk;
      const K128 key = valid ? src[p] : K128{0ull, 0ull};
      const uint32_t d = valid ? 255u - digit(key, shift) : 256u;  // invalid: own group
      for (int j = lane; j < 256; j += 32) whist[warp][j] = 0;
      __syncwarp();
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
      const uint32_t before = __popc(peers & lt);
      if (valid && before == 0) whist[warp][d] = __popc(peers);
      __syncthreads();
      // per digit: exclusive offsets across warps, and the tile total
      for (int dd = threadIdx.x; dd < 256; dd += NT) {
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const uint32_t c = whist[w][dd];
          whist[w][dd] = run;
          run += c;
        }
        ghist[dd] = run;  // tile total (ghist is free after the scan)
      }
      __syncthreads();
      if (valid) dst[runbase[d] + whist[warp][d] + before] = key;
      __syncthreads();
      for (int dd = threadIdx.x; dd < 256; dd += NT) runbase[dd] += ghist[dd];
      __syncthreads();
    }
    K128* t = src; src = dst; dst = t;
  }
  __syncthreads();
  for (int64_t p = threadIdx.x; p < kk; p += NT) out.put(s, p, src[p]);
}

// ------------------------------------------------------------------ host side
inline size_t al(size_t v) { return (v + 255) & ~(size_t)255; }

inline int64_t pow2_at_least(int64_t v) {
  int64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

template <class Src>
cudaError_t launch_small(const Src& src, int64_t nseg, int64_t L, int64_t kk, const Out& out,
                         uint32_t* flag, cudaStream_t st) {
  const int64_t p2 = pow2_at_least(std::max<int64_t>(L, 2));
  const size_t sm = (size_t)p2 * sizeof(K128);
  if (nseg == 0) return cudaSuccess;
  if (p2 <= 128) {
    f64_seg_small<64, Src><<<(unsigned)nseg, 64, sm, st>>>(src, (int)p2, kk, out, flag);
  } else if (p2 <= 1024) {
    f64_seg_small<256, Src><<<(unsigned)nseg, 256, sm, st>>>(src, (int)p2, kk, out, flag);
  } else {
    auto kern = f64_seg_small<1024, Src>;
    cudaError_t e = ensure_smem_attr((const void*)kern, sm);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)nseg, 1024, sm, st>>>(src, (int)p2, kk, out, flag);
  }
  return cudaGetLastError();
}

// Segmented top-kk over nseg segments of <= Lmax keys: small -> one CTA in
// smem; long -> select/compact to scratch a, then smem sort or LSD (a <-> b).
template <class Src>
cudaError_t seg_topk(const Src& src, int64_t nseg, int64_t Lmax, int64_t kk, const Out& out,
                     K128* a, K128* b, uint32_t* flag, cudaStream_t st) {
  if (Lmax <= SMALL_CAP) return launch_small(src, nseg, Lmax, kk, out, flag, st);
  f64_seg_select<512, Src><<<(unsigned)nseg, 512, 0, st>>>(src, kk, a, flag);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (kk <= SMALL_CAP) return launch_small(KeySrc{a, kk, kk}, nseg, kk, kk, out, nullptr, st);
  f64_lsd<512><<<(unsigned)nseg, 512, 0, st>>>(a, b, kk, out);
  return cudaGetLastError();
}

struct Plan {
  size_t pool = 0, s1 = 0, s2 = 0;  // pool keys; stage-1 / stage-2 long-segment scratch (x2 each)
  size_t total() const { return al(pool) + 2 * al(std::max(s1, s2)); }
};

inline Plan plan(int64_t m, int64_t n, int64_t k, int64_t b, int64_t kb) {
  Plan p;
  const int64_t s = (n + b - 1) / b;
  if (b == 1) {
    if (n > SMALL_CAP) p.s2 = (size_t)(m * k) * sizeof(K128);
    return p;
  }
  p.pool = (size_t)(m * b * kb) * sizeof(K128);
  if (kb > 16 && s > SMALL_CAP) p.s1 = (size_t)(m * b * kb) * sizeof(K128);
  if (b * kb > SMALL_CAP) p.s2 = (size_t)(m * k) * sizeof(K128);
  return p;
}

inline cudaError_t stage1_pool(const RowSrc& src, int64_t m, int64_t kb, K128* pool, K128* a, K128* b,
                               uint32_t* flag, cudaStream_t st) {
  if (kb <= 16) {
    dim3 grid((unsigned)((src.b + 255) / 256), (unsigned)std::min<int64_t>(m, 65535));
    const int t = kb <= 1 ? 1 : kb <= 2 ? 2 : kb <= 4 ? 4 : kb <= 8 ? 8 : 16;
    switch (t) {
      case 1: f64_s1_queue<1><<<grid, 256, 0, st>>>(src, m, kb, pool, flag); break;
      case 2: f64_s1_queue<2><<<grid, 256, 0, st>>>(src, m, kb, pool, flag); break;
      case 4: f64_s1_queue<4><<<grid, 256, 0, st>>>(src, m, kb, pool, flag); break;
      case 8: f64_s1_queue<8><<<grid, 256, 0, st>>>(src, m, kb, pool, flag); break;
      default: f64_s1_queue<16><<<grid, 256, 0, st>>>(src, m, kb, pool, flag); break;
    }
    return cudaGetLastError();
  }
  const int64_t s = (src.n + src.b - 1) / src.b;
  Out o{pool, nullptr, nullptr, kb};
  return seg_topk(src, m * src.b, s, kb, o, a, b, flag, st);
}

// pool (m x b*kb keys, bucket-major) -> compact (m x C) values/indices.
__global__ void f64_emit(RowSrc src, int64_t m, int64_t kb, int64_t C, const K128* __restrict__ pool,
                         uint64_t* __restrict__ vals, int64_t* __restrict__ idx) {
  const int64_t b = src.b, n = src.n;
  const int64_t total = m * b * kb;
  const int64_t q0 = n / b, r = n % b;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t qq = t % kb, rb = t / kb;
    const int64_t j = rb % b, row = rb / b;
    int64_t start, size, step;
    src.span(j, start, size, step);
    if (qq >= size) continue;
    int64_t off;
    if (kb <= q0) off = j * kb;
    else off = (src.layout == 0) ? (j * q0 + (j < r ? j : r)) : start;
    uint64_t bits;
    int64_t lab;
    decode(pool[t], bits, lab);
    vals[row * C + off + qq] = bits;
    idx[row * C + off + qq] = lab;
  }
}

struct Carve {
  uint8_t* p;
  K128* take(size_t bytes) {
    if (!bytes) return nullptr;
    K128* r = reinterpret_cast<K128*>(p);
    p += al(bytes);
    return r;
  }
};

}  // namespace f64

// ------------------------------------------------------------------ entry points (btk_api.cu)
size_t f64_workspace_bytes(int64_t m, int64_t n, int64_t k, int64_t b, int64_t kb) {
  return f64::plan(m, n, k, b, kb).total();
}

size_t f64_stage1_workspace_bytes(int64_t m, int64_t n, int64_t b, int64_t kb) {
  f64::Plan p = f64::plan(m, n, std::min<int64_t>(n, b * kb), b, kb);
  p.pool = (size_t)(m * b * kb) * sizeof(f64::K128);
  p.s2 = 0;
  if (b == 1 && n > f64::SMALL_CAP) p.s1 = (size_t)(m * kb) * sizeof(f64::K128);
  return p.total();
}

cudaError_t f64_approx_topk(const void* x, int64_t row_stride, int64_t m, int64_t n, int64_t k, int64_t b,
                            int64_t kb, int layout, void* out_vals, int64_t* out_idx, void* ws,
                            uint32_t* flag, cudaStream_t st) {
  using namespace f64;
  const Plan pl = plan(m, n, k, b, kb);
  Carve cv{static_cast<uint8_t*>(ws)};
  K128* pool = cv.take(pl.pool);
  const size_t sc = std::max(pl.s1, pl.s2);
  K128* a = cv.take(sc);
  K128* bb = cv.take(sc);
  RowSrc src{static_cast<const uint64_t*>(x), row_stride, n, b, layout};
  Out out{nullptr, static_cast<uint64_t*>(out_vals), out_idx, k};
  if (b == 1) return seg_topk(src, m, n, k, out, a, bb, flag, st);  // exact: one segment per row
  cudaError_t e = stage1_pool(src, m, kb, pool, a, bb, flag, st);
  if (e != cudaSuccess) return e;
  return seg_topk(KeySrc{pool, b * kb, b * kb}, m, b * kb, k, out, a, bb, nullptr, st);
}

cudaError_t f64_stage1(const void* x, int64_t row_stride, int64_t m, int64_t n, int64_t b, int64_t kb,
                       int layout, int64_t C, void* out_vals, int64_t* out_idx, void* ws, uint32_t* flag,
                       cudaStream_t st) {
  using namespace f64;
  Carve cv{static_cast<uint8_t*>(ws)};
  K128* pool = cv.take((size_t)(m * b * kb) * sizeof(K128));
  const size_t sc = (b == 1 && n > SMALL_CAP) ? (size_t)(m * kb) * sizeof(K128)
                                              : ((kb > 16 && (n + b - 1) / b > SMALL_CAP)
                                                     ? (size_t)(m * b * kb) * sizeof(K128) : 0);
  K128* a = cv.take(sc);
  K128* bb = cv.take(sc);
  RowSrc src{static_cast<const uint64_t*>(x), row_stride, n, b, layout};
  cudaError_t e = stage1_pool(src, m, kb, pool, a, bb, flag, st);
  if (e != cudaSuccess) return e;
  const int64_t total = m * b * kb;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 64));
  f64_emit<<<grid, 256, 0, st>>>(src, m, kb, C, pool, static_cast<uint64_t*>(out_vals), out_idx);
  return cudaGetLastError();
}

size_t f64_pairs_workspace_bytes(int64_t m, int64_t c, int64_t k) {
  if (c <= f64::SMALL_CAP) return 0;
  return 2 * f64::al((size_t)(m * k) * sizeof(f64::K128));
}

cudaError_t f64_topk_with_indices(const void* values, const int64_t* labels, int64_t m, int64_t c,
                                  int64_t k, void* out_vals, int64_t* out_idx, void* ws, uint32_t* flag,
                                  cudaStream_t st) {
  using namespace f64;
  Carve cv{static_cast<uint8_t*>(ws)};
  const size_t sc = c > SMALL_CAP ? (size_t)(m * k) * sizeof(K128) : 0;
  K128* a = cv.take(sc);
  K128* bb = cv.take(sc);
  Out out{nullptr, static_cast<uint64_t*>(out_vals), out_idx, k};
  return seg_topk(PairSrc{static_cast<const uint64_t*>(values), labels, c}, m, c, k, out, a, bb, flag, st);
}

}  // namespace btk
