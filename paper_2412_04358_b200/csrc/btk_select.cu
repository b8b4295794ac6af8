// K2: segmented exact top-kk over composite keys, emitted in canonical order.
//
// Restates reference exact.py:142-159 (topk_with_indices / _canonical_order)
// for the GPU: candidates of one segment (a row's Stage-1 survivors, or one
// bucket when k_b is large) are reduced to their kk largest composite keys,
// sorted descending.  Because comps are unique and their unsigned order is
// (value desc, index asc), "sort comps descending, take kk" IS the
// reference's two stable argsorts.
//
//   L <= SMALL_CAP : one CTA per segment, keys resident in shared memory,
//                    LSD radix sort (btk_sort.cuh), epilogue writes kk.
//   L >  SMALL_CAP : k2_select_compact (MSD radix select of the kk-th key
//                    with 256-bin smem histograms, then compaction), then
//                    the smem sort if kk fits, else k2_global_lsd (stable
//                    LSD passes through a global ping-pong buffer).
#include "btk_internal.h"
#include "btk_k2dev.cuh"
#include "btk_rank.cuh"
#include "btk_sort.cuh"

namespace btk {

// ---------------------------------------------------------------------------
// One CTA per segment of L <= NT*ITEMS keys: keys into shared memory, the
// bucketing/rank engine (btk_rank.cuh) finds the kk largest in order.
template <int DT, int NT, int ITEMS, bool DECODE, bool UNIQ>
__global__ void __launch_bounds__(NT) k2_small(const uint64_t* __restrict__ in, int64_t in_stride,
                                               int64_t L, int64_t kk, uint64_t* __restrict__ out_keys,
                                               void* __restrict__ out_vals,
                                               int64_t* __restrict__ out_idx, int64_t out_stride,
                                               CompGeo g, int lognb, const int* mask,
                                               int64_t mask_stride) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // let a programmatic dependent (the next call's Stage 1 with
  // BTK_INPUT_READY) start streaming; it waits before its first write
  asm volatile("griddepcontrol.launch_dependents;");
  uint64_t* sk = reinterpret_cast<uint64_t*>(smem_raw);
  uint8_t* aux = smem_raw + ((size_t)L * 8 + 127) / 128 * 128;
  const RankSmem S = rank_smem(sk, aux, L, kk, lognb, NT);
  const int64_t seg = blockIdx.x;
  if (mask && mask[seg * mask_stride] >= 0) return;  // row handled by the chunked path
  const uint64_t* src = in + seg * in_stride;
  for (int p = threadIdx.x; p < L; p += NT) sk[p] = src[p];
  __syncthreads();
  rank_select_sort<DT, NT, ITEMS, UNIQ>(S, (int)L, (int)kk, lognb, g.ib);
  // fewer than kk non-empty keys (only via empty slots): pad with 0 = "empty"
  for (int p = threadIdx.x; p < kk; p += NT) {
    const uint64_t c = rs_key(sk, S.inv[p]);
    if constexpr (DECODE) {
      emit<DT>(c, seg * out_stride + p, g, out_vals, out_idx);
    } else {
      out_keys[seg * out_stride + p] = c;
    }
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) k2_select_compact(const uint64_t* __restrict__ in,
                                                        int64_t in_stride, int64_t L, int64_t kk,
                                                        uint64_t* __restrict__ out,
                                                        int64_t out_stride, int nbits,
                                                        const int* mask, int64_t mask_stride) {
  const int64_t seg = blockIdx.x;
  if (mask && mask[seg * mask_stride] >= 0) return;
  uint32_t bad = 0;
  select_compact<NT>(CompSource{in + seg * in_stride}, L, kk, out + seg * out_stride, nbits, bad);
}

// Exact top-kk composite keys of every bucket of raw score rows, unsorted
// (0 = empty slot): one CTA per (row, bucket), buckets laid out as in the
// reference (interleaved j + b*t / contiguous slices, core.py:124-147).
template <int DT, int NT>
__global__ void __launch_bounds__(NT) k2_select_raw(const void* __restrict__ x, int64_t row_stride, int64_t n,
                                                    int64_t nb, int layout, int64_t kk,
                                                    uint64_t* __restrict__ out, CompGeo g, uint32_t* flag) {
  const int64_t seg = blockIdx.x, row = seg / nb, j = seg - row * nb;
  int64_t start, size, step;
  if (layout == 0) {
    const int64_t q = n / nb, r = n % nb;
    start = j; size = q + (j < r ? 1 : 0); step = nb;
  } else {
    start = (j * n + nb - 1) / nb;
    size = ((j + 1) * n + nb - 1) / nb - start;
    step = 1;
  }
  uint32_t bad = 0;
  const RawSource<DT> src{static_cast<const uint8_t*>(x) + row * row_stride * (VT<DT>::W / 8), start, step, g};
  select_compact<NT>(src, size, kk, out + seg * kk, g.nbits, bad);
  if (__syncthreads_or(bad) && threadIdx.x == 0 && flag) atomicOr(flag, 1u);
}

// ---------------------------------------------------------------------------
// Stable LSD sort of kk keys per segment through a global ping-pong buffer,
// one CTA per segment; the epilogue writes the sorted keys out.
template <int DT, int NT, int ITEMS, bool DECODE>
__global__ void __launch_bounds__(NT) k2_global_lsd(uint64_t* __restrict__ A, uint64_t* __restrict__ B,
                                                    int64_t stride_a, int64_t stride_b, int64_t kk,
                                                    uint64_t* __restrict__ out_keys,
                                                    void* __restrict__ out_vals,
                                                    int64_t* __restrict__ out_idx,
                                                    int64_t out_stride, CompGeo g,
                                                    const int* mask, int64_t mask_stride) {
  const int64_t seg = blockIdx.x;
  if (mask && mask[seg * mask_stride] >= 0) return;
  const uint64_t* src = global_lsd<NT, ITEMS>(A + seg * stride_a, B + seg * stride_b, kk, g.nbits);
  for (int64_t p = threadIdx.x; p < kk; p += NT) {
    if constexpr (DECODE) {
      emit<DT>(src[p], seg * out_stride + p, g, out_vals, out_idx);
    } else {
      out_keys[seg * out_stride + p] = src[p];
    }
  }
}

// ---------------------------------------------------------------------------
template <int DT>
__global__ void k2_decode(const uint64_t* __restrict__ in, int64_t in_stride, int64_t nseg,
                          int64_t kk, void* __restrict__ out_vals, int64_t* __restrict__ out_idx,
                          int64_t out_stride, CompGeo g) {
  const int64_t total = nseg * kk;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t seg = t / kk, p = t - seg * kk;
    emit<DT>(in[seg * in_stride + p], seg * out_stride + p, g, out_vals, out_idx);
  }
}

// ---------------------------------------------------------------------------
// Host dispatch.
template <int DT, int NT, int ITEMS, bool DECODE>
static cudaError_t launch_small(const K2Args& a, cudaStream_t st) {
  auto kern = a.unique ? k2_small<DT, NT, ITEMS, DECODE, true> : k2_small<DT, NT, ITEMS, DECODE, false>;
  const int lognb = rank_lognb(a.L);
  const size_t sm = ((size_t)a.L * 8 + 127) / 128 * 128 + rank_aux_bytes(NT, lognb, a.kk, a.L);
  cudaError_t e = ensure_smem_attr((const void*)kern, sm);
  if (e != cudaSuccess) return e;
  if (a.nseg == 0) return cudaSuccess;
  kern<<<(unsigned)a.nseg, NT, sm, st>>>(a.in, a.in_stride, a.L, a.kk, a.out_keys, a.out_vals,
                                         a.out_idx, a.out_stride, a.geo, lognb, a.mask, a.mask_stride);
  return cudaGetLastError();
}

template <int DT, bool DECODE>
static cudaError_t run_small(const K2Args& a, cudaStream_t st) {
  const int64_t L = a.L;
  if (L <= 64) return launch_small<DT, 64, 1, DECODE>(a, st);
  if (L <= 256) return launch_small<DT, 128, 2, DECODE>(a, st);
  if (L <= 1024) return launch_small<DT, 256, 4, DECODE>(a, st);
  if (L <= 4096) return launch_small<DT, 512, 8, DECODE>(a, st);
  return launch_small<DT, 512, 32, DECODE>(a, st);
}

template <int DT, bool DECODE>
static cudaError_t run_k2_t(const K2Args& a, cudaStream_t st) {
  if (a.L <= K2_SMALL_CAP) return run_small<DT, DECODE>(a, st);
  // long segments
  if (a.scratch_a == nullptr || a.scratch_b == nullptr) return cudaErrorInvalidValue;
  const int64_t sa = a.scratch_a_stride ? a.scratch_a_stride : a.kk;
  const int64_t sb = a.scratch_b_stride ? a.scratch_b_stride : a.kk;
  k2_select_compact<1024><<<(unsigned)a.nseg, 1024, 0, st>>>(a.in, a.in_stride, a.L, a.kk,
                                                             a.scratch_a, sa, a.geo.nbits, a.mask,
                                                             a.mask_stride);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (a.kk <= K2_SMALL_CAP) {
    K2Args b = a;
    b.in = a.scratch_a;
    b.in_stride = sa;
    b.L = a.kk;
    return run_small<DT, DECODE>(b, st);
  }
  k2_global_lsd<DT, 512, 8, DECODE><<<(unsigned)a.nseg, 512, 0, st>>>(
      a.scratch_a, a.scratch_b, sa, sb, a.kk, a.out_keys, a.out_vals, a.out_idx, a.out_stride, a.geo,
      a.mask, a.mask_stride);
  return cudaGetLastError();
}

template <int DT, int NT>
static void launch_select_raw(const void* x, int64_t row_stride, int64_t m, int64_t n, int64_t nb, int layout,
                              int64_t kk, uint64_t* out, CompGeo g, uint32_t* flag, cudaStream_t st) {
  k2_select_raw<DT, NT><<<(unsigned)(m * nb), NT, 0, st>>>(x, row_stride, n, nb, layout, kk, out, g, flag);
}

template <int DT>
static void select_raw_dt(const void* x, int64_t row_stride, int64_t m, int64_t n, int64_t nb, int layout,
                          int64_t kk, uint64_t* out, CompGeo g, uint32_t* flag, cudaStream_t st) {
  if (n / nb >= 16384) launch_select_raw<DT, 1024>(x, row_stride, m, n, nb, layout, kk, out, g, flag, st);
  else launch_select_raw<DT, 256>(x, row_stride, m, n, nb, layout, kk, out, g, flag, st);
}

cudaError_t run_select_raw(int dtype, const void* x, int64_t row_stride, int64_t m, int64_t n, int64_t nb,
                           int layout, int64_t kk, uint64_t* out, CompGeo g, uint32_t* flag, cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  if (m * nb > 0x7FFFFFFFll) return cudaErrorInvalidValue;
  switch (dtype) {
    case F32: select_raw_dt<F32>(x, row_stride, m, n, nb, layout, kk, out, g, flag, st); break;
    case BF16: select_raw_dt<BF16>(x, row_stride, m, n, nb, layout, kk, out, g, flag, st); break;
    case F16: select_raw_dt<F16>(x, row_stride, m, n, nb, layout, kk, out, g, flag, st); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t run_k2(int dtype, bool decode, const K2Args& a, cudaStream_t st) {
  switch (dtype) {
    case F32: return decode ? run_k2_t<F32, true>(a, st) : run_k2_t<F32, false>(a, st);
    case BF16: return decode ? run_k2_t<BF16, true>(a, st) : run_k2_t<BF16, false>(a, st);
    case F16: return decode ? run_k2_t<F16, true>(a, st) : run_k2_t<F16, false>(a, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t run_decode(int dtype, const uint64_t* in, int64_t in_stride, int64_t nseg, int64_t kk,
                       void* out_vals, int64_t* out_idx, int64_t out_stride, CompGeo g,
                       cudaStream_t st) {
  int64_t total = nseg * kk;
  if (total == 0) return cudaSuccess;
  unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 32);
  switch (dtype) {
    case F32: k2_decode<F32><<<grid, 256, 0, st>>>(in, in_stride, nseg, kk, out_vals, out_idx, out_stride, g); break;
    case BF16: k2_decode<BF16><<<grid, 256, 0, st>>>(in, in_stride, nseg, kk, out_vals, out_idx, out_stride, g); break;
    case F16: k2_decode<F16><<<grid, 256, 0, st>>>(in, in_stride, nseg, kk, out_vals, out_idx, out_stride, g); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace btk
