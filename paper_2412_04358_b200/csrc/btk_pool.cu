// Chunked Stage 2 for large Stage-1 pools (cfg5: 131072 survivors per row,
// k = 65536): the exact canonical top-k of each row's pool without a
// global radix select or a global sort.
//
// Restates reference exact.py:130-159 (topk_with_indices: stable argsort
// by index, then by -value, take k) for composite keys, whose unsigned
// order is that order (btk_common.cuh).
//
//   s1_vec<HIST>   (btk_fused_impl.cuh) writes the pool AND a per-row
//                  histogram of the survivors' coarse bins (top POOL_HBITS
//                  bits of the key), so planning needs no extra pool read.
//   pool_scatter   one CTA per row: descending exclusive scan of the
//                  histogram -> threshold bin (the one holding the k-th
//                  key) and chunks of whole bins starting at multiples of
//                  POOL_HALF keys (chunk of bin = excl / POOL_HALF), then
//                  ONE read of the pool scattering every key of a selected
//                  bin into its chunk's slice of the chunk buffer.  The
//                  chunk slices are laid out in output order, so a chunk's
//                  offset in the buffer is its offset in the output row.
//   pool_sort      one CTA per (row, chunk): the chunk's <= 2*POOL_HALF
//                  keys in shared memory, LSD radix sort (4-bit digits,
//                  register counters + block scan ranking; only the bits
//                  that vary inside the chunk are passed over), then the
//                  first min(count, k - offset) keys are decoded and
//                  written.
//
// A row whose selected bins hold more than POOL_HALF keys in one bin
// (massive ties) is marked in its chunk table (n = -1) and takes the
// radix-select + sort fallback (btk_select.cu) for that row only.
//
// Bytes per row (cfg5, bf16): pool 1 MB written by s1_vec, read once here;
// chunk buffer ~0.55 MB written and read once; output 0.64 MB.
#include <cstdlib>

#include "btk_internal.h"

namespace btk {
namespace {

constexpr int NBINS = 1 << POOL_HBITS;
constexpr int SC_NT = 1024;            // pool_scatter threads
constexpr int SO_NT = 1024;            // pool_sort threads
constexpr int SO_ITEMS = 16;           // keys per thread (blocked)
constexpr int SO_CAP = SO_NT * SO_ITEMS;  // 16384 = 2 * POOL_HALF
static_assert(SO_CAP >= 2 * POOL_HALF, "chunk capacity");

__host__ __device__ __forceinline__ int pad_of(int p) { return p + ((p >> 4) << 1); }  // 16 B pad per 128 B

// ------------------------------------------------------------------ plan + scatter
__global__ void __launch_bounds__(SC_NT) pool_scatter(const uint64_t* __restrict__ pool, int64_t P,
                                                      const uint32_t* __restrict__ hist, int64_t k,
                                                      int hshift, uint64_t* __restrict__ buf,
                                                      int64_t buf_stride, ChunkTab* __restrict__ tab) {
  __shared__ uint32_t excl[NBINS];  // descending exclusive prefix per bin
  __shared__ uint32_t wsum[SC_NT / 32];
  __shared__ int cstart[POOL_MAXC + 2];
  __shared__ uint32_t cursor[POOL_MAXC];
  __shared__ int s_bad, s_nch, s_total;
  const int64_t row = blockIdx.x;
  const uint32_t* h = hist + row * NBINS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int PER = NBINS / SC_NT;  // 8 bins per thread, in descending bin order
  uint32_t c[PER], sum = 0;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    c[i] = h[NBINS - 1 - (tid * PER + i)];
    sum += c[i];
  }
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[warp] = incl;
  if (tid < POOL_MAXC + 2) cstart[tid] = 0x7FFFFFFF;
  if (tid < POOL_MAXC) cursor[tid] = 0u;
  if (tid == 0) { s_bad = 0; s_nch = 0; s_total = 0; }
  __syncthreads();
  uint32_t wbase = 0;
  for (int w = 0; w < warp; ++w) wbase += wsum[w];
  uint32_t run = wbase + incl - sum;
  bool bad = false;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int bin = NBINS - 1 - (tid * PER + i);
    excl[bin] = run;
    if (run < (uint32_t)k && c[i]) {  // a selected bin
      bad |= c[i] > (uint32_t)POOL_HALF;
      const int ch = (int)(run / POOL_HALF);
      if (ch >= POOL_MAXC) bad = true;
      else atomicMin(&cstart[ch], (int)run);
      if (run + c[i] >= (uint32_t)k) {  // the threshold bin (holds the k-th key)
        s_nch = ch + 1;
        s_total = (int)(run + c[i]);
      }
    }
    run += c[i];
  }
  if (bad) s_bad = 1;
  __syncthreads();
  ChunkTab* T = tab + row;
  if (s_bad || s_nch == 0) {  // fallback row (or fewer than k keys: never for validated shapes)
    if (tid == 0) T->n = -1;
    return;
  }
  const int nch = s_nch;
  if (tid == 0) {
    cstart[nch] = s_total;
    for (int ch = nch - 1; ch >= 0; --ch) cstart[ch] = min(cstart[ch], cstart[ch + 1]);  // empty chunks
    T->n = nch;
    for (int ch = 0; ch <= nch; ++ch) T->start[ch] = cstart[ch];
  }
  __syncthreads();
  // one read of the pool: every key of a selected bin goes to its chunk
  const uint64_t* src = pool + row * P;
  uint64_t* dst = buf + row * buf_stride;
  for (int64_t p0 = 0; p0 < P; p0 += SC_NT) {
    const int64_t p = p0 + tid;
    const uint64_t key = p < P ? src[p] : 0ull;
    int ch = -1;
    if (key) {
      const uint32_t e = excl[(uint32_t)(key >> hshift)];
      if (e < (uint32_t)k) ch = (int)(e / POOL_HALF);
    }
    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, ch);
    if (ch >= 0) {
      const int leader = __ffs(peers) - 1;
      uint32_t base = 0;
      if (lane == leader) base = atomicAdd(&cursor[ch], (uint32_t)__popc(peers));
      base = __shfl_sync(peers, base, leader);
      dst[cstart[ch] + base + __popc(peers & lanemask_lt())] = key;
    }
  }
}

// ------------------------------------------------------------------ chunk sort
template <int DT>
__device__ __forceinline__ void emit_key(uint64_t c, int64_t pos, const CompGeo& g, void* out_vals,
                                         int64_t* out_idx) {
  uint32_t bits;
  int64_t idx;
  decode_comp<DT>(c, g, bits, idx);
  store_bits<DT>(out_vals, pos, bits);
  out_idx[pos] = idx;
}

// 16 bins x 8-bit counts in two u64 (bins 0-7 / 8-15)
__device__ __forceinline__ void cnt_add(uint64_t& lo, uint64_t& hi, uint32_t d) {
  const uint64_t one = 1ull << ((d & 7u) * 8u);
  if (d < 8u) lo += one; else hi += one;
}
__device__ __forceinline__ uint32_t cnt_get(uint64_t lo, uint64_t hi, uint32_t d) {
  return (uint32_t)(((d < 8u ? lo : hi) >> ((d & 7u) * 8u)) & 0xFFull);
}

template <int DT>
__global__ void __launch_bounds__(SO_NT, 1) pool_sort(const uint64_t* __restrict__ buf, int64_t buf_stride,
                                                      const ChunkTab* __restrict__ tab, int64_t k,
                                                      int nbits, CompGeo g, void* __restrict__ out_vals,
                                                      int64_t* __restrict__ out_idx) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint64_t* sk = reinterpret_cast<uint64_t*>(smem_raw);                              // padded keys
  uint16_t* tbase = reinterpret_cast<uint16_t*>(smem_raw + (size_t)pad_of(SO_CAP) * 8);  // [SO_NT][16]
  __shared__ uint32_t wsum[SO_NT / 32][8];
  __shared__ uint32_t dbase[16];
  __shared__ unsigned long long s_or;
  const int64_t row = blockIdx.y;
  const int ch = blockIdx.x;
  const ChunkTab* T = tab + row;
  const int nch = T->n;
  if (ch >= nch) return;  // no such chunk (or a fallback row: n = -1)
  const int start = T->start[ch], cnt = T->start[ch + 1] - start;
  const int keep = (int)min((int64_t)cnt, k - start);
  if (keep <= 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t* src = buf + row * buf_stride + start;
  // load (coalesced), OR of differences to find the varying bits
  const uint64_t k0 = src[0];
  uint64_t diff = 0;
  for (int p = tid; p < SO_CAP; p += SO_NT) {
    const uint64_t key = p < cnt ? src[p] : 0ull;  // 0 pads sort last (descending)
    if (p < cnt) diff |= key ^ k0;
    sk[pad_of(p)] = key;
  }
  if (tid == 0) s_or = 0ull;
  __syncthreads();
#pragma unroll
  for (int o = 16; o; o >>= 1) diff |= __shfl_xor_sync(0xFFFFFFFFu, diff, o);
  if (lane == 0 && diff) atomicOr(&s_or, (unsigned long long)diff);
  __syncthreads();
  const uint64_t vary = s_or;
  for (int shift = 1; shift < nbits; shift += 4) {
    if (((vary >> shift) & 0xFull) == 0ull) continue;  // digit constant over the chunk: identity pass
    // phase 1: digit counts of this thread's SO_ITEMS consecutive keys
    uint64_t lo = 0, hi = 0;
#pragma unroll
    for (int i = 0; i < SO_ITEMS; i += 2) {
      const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(&sk[pad_of(tid * SO_ITEMS + i)]);
      cnt_add(lo, hi, 15u - (uint32_t)((v.x >> shift) & 0xFull));
      cnt_add(lo, hi, 15u - (uint32_t)((v.y >> shift) & 0xFull));
    }
    // 16 counts -> 8 words of 2 x 16-bit fields; warp inclusive scan
    auto own = [&](int q) -> uint32_t {
      const uint64_t src64 = q < 4 ? lo : hi;
      const int b0 = (q & 3) * 16;
      return (uint32_t)((src64 >> b0) & 0xFF) | ((uint32_t)((src64 >> (b0 + 8)) & 0xFF) << 16);
    };
    uint32_t w[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) w[q] = own(q);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, w[q], o);
        if (lane >= o) w[q] += t;
      }
    }
    if (lane == 31) {
#pragma unroll
      for (int q = 0; q < 8; ++q) wsum[warp][q] = w[q];
    }
    __syncthreads();
    if (tid < 8) {  // exclusive scan over warps, per word; block totals per digit
      uint32_t r = 0;
      for (int ww = 0; ww < SO_NT / 32; ++ww) {
        const uint32_t v = wsum[ww][tid];
        wsum[ww][tid] = r;
        r += v;
      }
      dbase[2 * tid] = r & 0xFFFFu;
      dbase[2 * tid + 1] = r >> 16;
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t acc = 0;
#pragma unroll
      for (int d = 0; d < 16; ++d) { const uint32_t v = dbase[d]; dbase[d] = acc; acc += v; }
    }
    __syncthreads();
    // this thread's first rank per digit (digit-major, thread, item order: stable)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t ex = w[q] - own(q) + wsum[warp][q];
      tbase[tid * 16 + 2 * q] = (uint16_t)(dbase[2 * q] + (ex & 0xFFFFu));
      tbase[tid * 16 + 2 * q + 1] = (uint16_t)(dbase[2 * q + 1] + (ex >> 16));
    }
    // phase 2: keys to registers, then scatter in place
    uint64_t key[SO_ITEMS];
#pragma unroll
    for (int i = 0; i < SO_ITEMS; i += 2) {
      const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(&sk[pad_of(tid * SO_ITEMS + i)]);
      key[i] = v.x;
      key[i + 1] = v.y;
    }
    __syncthreads();
    lo = hi = 0;
#pragma unroll
    for (int i = 0; i < SO_ITEMS; ++i) {
      const uint32_t d = 15u - (uint32_t)((key[i] >> shift) & 0xFull);
      const int r = (int)tbase[tid * 16 + d] + (int)cnt_get(lo, hi, d);
      cnt_add(lo, hi, d);
      sk[pad_of(r)] = key[i];
    }
    __syncthreads();
  }
  for (int q = tid; q < keep; q += SO_NT)
    emit_key<DT>(sk[pad_of(q)], (int64_t)row * k + start + q, g, out_vals, out_idx);
}

}  // namespace

bool pool_chunked_ok(const Problem& p) {
  if (!stage1_vec_supported(p)) return false;
  if (p.b * p.kb <= K2_SMALL_CAP) return false;      // small pools: K2 in one CTA
  if (p.k > (int64_t)(POOL_MAXC - 1) * POOL_HALF) return false;
  if (p.b * p.kb >= (int64_t(1) << 31)) return false;
  return std::getenv("BTK_POOL_CHUNKED") == nullptr || std::atoi(std::getenv("BTK_POOL_CHUNKED")) != 0;
}

static size_t al(size_t v) { return (v + 255) & ~(size_t)255; }

size_t pool_chunked_bytes(const Problem& p) {
  return al((size_t)p.m * NBINS * 4) + al((size_t)p.m * sizeof(ChunkTab)) +
         al((size_t)p.m * (p.k + POOL_HALF) * 8);
}

template <int DT>
static cudaError_t sort_launch(const Problem& p, const uint64_t* buf, int64_t bs, const ChunkTab* tab,
                               void* out_vals, int64_t* out_idx, cudaStream_t st) {
  const size_t sm = (size_t)pad_of(SO_CAP) * 8 + (size_t)SO_NT * 16 * 2;
  auto kern = pool_sort<DT>;
  cudaError_t e = ensure_smem_attr((const void*)kern, sm);
  if (e != cudaSuccess) return e;
  const int maxc = (int)std::min<int64_t>(POOL_MAXC, (p.k + POOL_HALF - 1) / POOL_HALF + 1);
  kern<<<dim3((unsigned)maxc, (unsigned)p.m), SO_NT, sm, st>>>(buf, bs, tab, p.k, p.geo.nbits, p.geo,
                                                                out_vals, out_idx);
  return cudaGetLastError();
}

// ws layout: hist | tab | chunk buffer.  The pool (m x b*kb) is the caller's.
cudaError_t run_pool_chunked(const Problem& p, uint64_t* pool, void* ws, void* out_vals,
                             int64_t* out_idx, cudaStream_t st) {
  uint8_t* w = static_cast<uint8_t*>(ws);
  uint32_t* hist = reinterpret_cast<uint32_t*>(w);
  w += al((size_t)p.m * NBINS * 4);
  ChunkTab* tab = reinterpret_cast<ChunkTab*>(w);
  w += al((size_t)p.m * sizeof(ChunkTab));
  uint64_t* buf = reinterpret_cast<uint64_t*>(w);
  const int64_t bs = p.k + POOL_HALF;
  const int64_t P = p.b * p.kb;
  cudaError_t e = cudaMemsetAsync(hist, 0, (size_t)p.m * NBINS * 4, st);
  if (e != cudaSuccess) return e;
  e = run_stage1_vec(p, pool, st, hist);
  if (e != cudaSuccess) return e;
  pool_scatter<<<(unsigned)p.m, SC_NT, 0, st>>>(pool, P, hist, p.k, p.geo.nbits - POOL_HBITS, buf, bs, tab);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  switch (p.dtype) {
    case F32: e = sort_launch<F32>(p, buf, bs, tab, out_vals, out_idx, st); break;
    case BF16: e = sort_launch<BF16>(p, buf, bs, tab, out_vals, out_idx, st); break;
    default: e = sort_launch<F16>(p, buf, bs, tab, out_vals, out_idx, st); break;
  }
  if (e != cudaSuccess) return e;
  // fallback rows (tab[row].n == -1): radix select + sort over the pool;
  // scratch a = the chunk buffer (stride k + POOL_HALF), scratch b = the pool
  K2Args a{};
  a.in = pool; a.in_stride = P; a.nseg = p.m; a.L = P; a.kk = p.k;
  a.out_vals = out_vals; a.out_idx = out_idx; a.out_stride = p.k;
  a.geo = p.geo; a.scratch_a = buf; a.scratch_b = pool;
  a.scratch_a_stride = bs; a.scratch_b_stride = P;
  a.mask = &tab[0].n;
  a.mask_stride = (int64_t)(sizeof(ChunkTab) / sizeof(int));
  return run_k2(p.dtype, true, a, st);
}

}  // namespace btk
