// Generic Stage 1: per-bucket top-k_b for any layout / raggedness / dtype.
//
// Restates reference approx.py:112-173 + 208-242 (index map, cube gather,
// top-k_b per bucket, ragged keep-mask) without materialising the cube:
// one thread owns one (row, bucket), walks the bucket's positions in
// increasing index order and keeps a register-resident insertion queue of
// composite keys.  A strict ">" test suffices (the scan order makes any
// later tie lose), mirroring the reference's "first maximum" argmax.
//
// This is the universal path (contiguous layout, ragged shapes, odd
// strides).  Interleaved shapes inside the fused envelope take
// btk_fused.cu instead.
#include "btk_fused_impl.cuh"  // Queue, vector loads and unpacking (namespace fz)

namespace btk {

__device__ __forceinline__ void bucket_span(const Problem& p, int64_t j, int64_t& start,
                                            int64_t& size, int64_t& step) {
  if (p.layout == 0) {
    const int64_t q = p.n / p.b, r = p.n % p.b;
    start = j;
    size = q + (j < r ? 1 : 0);
    step = p.b;
  } else {
    start = (j * p.n + p.b - 1) / p.b;
    const int64_t end = ((j + 1) * p.n + p.b - 1) / p.b;
    size = end - start;
    step = 1;
  }
}

template <int DT>
__device__ __forceinline__ uint64_t elem_comp(const Problem& p, const void* row, int64_t idx,
                                              bool& bad) {
  const uint32_t bits = load_bits<DT>(row, idx);
  bad |= nonfinite<DT>(bits);
  return make_comp(vkey<DT>(bits), (uint32_t)idx, is_negzero<DT>(bits), p.geo);
}

template <int DT, int KB>
__global__ void __launch_bounds__(256) s1_generic(Problem p, uint64_t* __restrict__ pool) {
  const int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int64_t P = p.b * p.kb;
  bool bad = false;
  for (int64_t row = blockIdx.y; row < p.m; row += gridDim.y) {
    if (j < p.b) {
      const void* xr = static_cast<const uint8_t*>(p.x) +
                       row * p.row_stride * (VT<DT>::W / 8);
      int64_t start, size, step;
      bucket_span(p, j, start, size, step);
      uint64_t q[KB];
#pragma unroll
      for (int i = 0; i < KB; ++i) q[i] = 0ull;
      for (int64_t t = 0; t < size; ++t) {
        const uint64_t c = elem_comp<DT>(p, xr, start + t * step, bad);
        if (c > q[KB - 1]) {
#pragma unroll
          for (int i = KB - 1; i > 0; --i) q[i] = (c > q[i - 1]) ? q[i - 1] : (c > q[i] ? c : q[i]);
          q[0] = (c > q[0]) ? c : q[0];
        }
      }
      uint64_t* dst = pool + row * P + j * p.kb;
#pragma unroll
      for (int i = 0; i < KB; ++i)
        if (i < p.kb) dst[i] = q[i];
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0 && p.flag) atomicOr(p.flag, 1u);
}

template <int DT>
__global__ void s1_emit(Problem p, const uint64_t* __restrict__ pool, int64_t C,
                        void* __restrict__ out_vals, int64_t* __restrict__ out_idx) {
  const int64_t total = p.m * p.b * p.kb;
  const int64_t q0 = p.n / p.b, r = p.n % p.b;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t qq = t % p.kb;
    const int64_t rb = t / p.kb;
    const int64_t j = rb % p.b, row = rb / p.b;
    int64_t start, size, step;
    bucket_span(p, j, start, size, step);
    if (qq >= size) continue;
    // closed-form bucket offset of sum_{j'<j} min(kb, size_j') (core.py:155-158)
    int64_t off;
    if (p.kb <= q0) off = j * p.kb;
    else off = (p.layout == 0) ? (j * q0 + (j < r ? j : r)) : start;
    uint32_t bits;
    int64_t idx;
    decode_comp<DT>(pool[t], p.geo, bits, idx);
    store_bits<DT>(out_vals, row * C + off + qq, bits);
    out_idx[row * C + off + qq] = idx;
  }
}

// ---------------------------------------------------------------------------
// Contiguous layout (bucket j = [ceil(jn/b), ceil((j+1)n/b)), reference
// core.py:124-147, approx.py:121-124): a bucket is a dense slice, so one
// WARP owns one (row, bucket).  Lane l streams vectors l, l+32, ... of the
// slice with 128-bit loads (coalesced: a warp instruction reads 512
// consecutive bytes), keeping a register queue of its top k_b (strict ">"
// in increasing index order = first maximum); the 32 queues then merge by
// k_b rounds of a warp max over composite keys (unique, canonical order).
// Slices that do not start/end on a 16-byte boundary take scalar loads.
template <int DT, int KB, int U>
__global__ void __launch_bounds__(256, (U <= 4 ? 4 : 2)) s1_contig(Problem p, uint64_t* __restrict__ pool, int G, int early) {
  constexpr int V = 16 / (VT<DT>::W / 8);
  constexpr int ESZ = VT<DT>::W / 8;
  const int lane = threadIdx.x & 31, gl = lane % G, per_warp = 32 / G;
  const int64_t P = p.b * p.kb;
  const int64_t tasks = p.m * p.b;
  // programmatic dependent launch: with BTK_INPUT_READY the slices are
  // streamed while the previous launch drains; the first pool write waits
  fz::pdl_trigger();
  if (!early) fz::pdl_wait();
  uint32_t bad = 0;
  // uniform buckets (b | n) and < 2^32 tasks: 32-bit index math, no 64-bit
  // divisions per bucket (they cost more than a bucket's loads)
  const bool uni = (p.n % p.b) == 0 && tasks < (int64_t(1) << 32) && p.b < (int64_t(1) << 31);
  const uint32_t b32 = (uint32_t)p.b, bsz = (uint32_t)(p.n / p.b);
  for (int64_t t0 = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * per_warp; t0 < tasks;
       t0 += (int64_t)gridDim.x * 8 * per_warp) {
    const int64_t task = t0 + lane / G;  // this lane group's (row, bucket)
    uint64_t best[KB];  // this lane's top k_b composite keys, descending
#pragma unroll
    for (int z = 0; z < KB; ++z) best[z] = 0ull;
    int64_t row = 0, j = 0;
    if (task < tasks) {
      int64_t start, size, step;
      if (uni) {
        const uint32_t r32 = (uint32_t)task / b32;
        row = r32;
        j = (uint32_t)task - r32 * b32;
        start = (int64_t)((uint32_t)j * bsz);
        size = bsz;
      } else {
        row = task / p.b;
        j = task - row * p.b;
        bucket_span(p, j, start, size, step);
      }
      const uint8_t* xr = static_cast<const uint8_t*>(p.x) + row * p.row_stride * ESZ;
      const bool vec = ((reinterpret_cast<uintptr_t>(xr) + start * ESZ) & 15) == 0 && (size % V) == 0 &&
                       size / V < 0xFFFF;
      if (vec) {
        // the lane's vectors as V sub-streams (one per element slot), each
        // with the packed / float queue of the fused scanners; the code of a
        // vector is its ordinal in the slice, so idx = start + code*V + slot
        const int64_t nv = size / V;
        const uint8_t* base = xr + start * ESZ;
        fz::Scanner<DT, KB> sc;
        sc.init();
        for (int64_t v0 = gl; v0 < nv; v0 += (int64_t)G * U) {
          uint4 w[U];
#pragma unroll
          for (int u = 0; u < U; ++u)
            w[u] = (v0 + G * u < nv) ? fz::ldg_stream(base + (v0 + G * u) * 16) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (v0 + G * u < nv) sc.row(w[u], (int)(v0 + G * u));
        }
        bad |= sc.nonfinite() ? 1u : 0u;
        // each_comp indexes code*V + slot from the slice start; the slice may
        // start at any element (row bases need not be 16-byte aligned), so
        // shift the index field by `start` (comp - 2*start: the field holds
        // IMAX - idx and never borrows into the value bits)
        const uint64_t shift_start = (uint64_t)start << 1;
        sc.each_comp(0, V, 0, p.geo, [&](int64_t, int, uint64_t c) {
          if (c) fz::comp_push<KB>(best, c - shift_start);
        });
      } else {
        fz::Queue<KB> q;
        q.init();
        for (int64_t t = gl; t < size; t += G) {
          const uint32_t bits = load_bits<DT>(xr, start + t);
          bad |= nonfinite<DT>(bits) ? 1u : 0u;
          float f;
          if constexpr (DT == F32) f = __uint_as_float(bits);
          else if constexpr (DT == BF16) f = __uint_as_float(bits << 16);
          else f = __half2float(__ushort_as_half((unsigned short)bits));
          q.push(f, (int)(start + t));
        }
#pragma unroll
        for (int z = 0; z < KB; ++z) best[z] = fz::comp_of<DT>(q.v[z], q.t[z], 0, 1, p.geo);  // idx = t
      }
    }
    // group merge: k_b rounds of a max over the group lanes' heads (xor
    // offsets < G stay inside the aligned group)
    int head = 0;
#pragma unroll
    for (int z = 0; z < KB; ++z) {
      uint64_t mine = 0ull;
#pragma unroll
      for (int i = 0; i < KB; ++i) mine = (i == head) ? best[i] : mine;
      uint64_t top = mine;
      for (int o = G >> 1; o; o >>= 1) {
        const uint64_t other = __shfl_xor_sync(0xFFFFFFFFu, top, o);
        top = other > top ? other : top;
      }
      if (top != 0ull && mine == top) ++head;  // comps are unique: one owner
      if (early && z == 0) fz::pdl_wait();  // the previous launch may still read the pool
      if (gl == 0 && task < tasks && z < p.kb) pool[row * P + j * p.kb + z] = top;
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0 && p.flag) atomicOr(p.flag, 1u);
}

template <int DT, int KB>
static cudaError_t launch_contig(const Problem& p, uint64_t* pool, cudaStream_t st) {
  // lanes per bucket: each lane streams >= 64 vectors of its bucket (the
  // per-bucket merge is amortised; measured at cfg3-contiguous: 16 -> 4.8,
  // 32 -> 4.9, 64 -> 5.1, 128 -> 4.6 TB/s)
  const int V = 16 / (VT<DT>::W / 8);
  const int64_t nv = (p.n / p.b) / V;
  const int vpl = fz::env_int("BTK_CONTIG_VPL", 64);  // min vectors per lane
  int G = 1;
  while (G < 32 && nv / (2 * G) >= vpl) G *= 2;
  const int64_t blocks = (p.m * p.b + 8 * (32 / G) - 1) / (8 * (32 / G));
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(blocks, 148 * 16));
  const int early = (p.flags & 1u) && fz::pdl_enabled() ? 1 : 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = fz::pdl_enabled() ? 1 : 0;
  if (fz::env_int("BTK_CONTIG_U", 4) == 8) return cudaLaunchKernelEx(&cfg, s1_contig<DT, KB, 8>, p, pool, G, early);
  return cudaLaunchKernelEx(&cfg, s1_contig<DT, KB, 4>, p, pool, G, early);
}

template <int DT>
static cudaError_t contig_t(const Problem& p, uint64_t* pool, cudaStream_t st) {
  if (p.kb <= 1) return launch_contig<DT, 1>(p, pool, st);
  if (p.kb <= 2) return launch_contig<DT, 2>(p, pool, st);
  if (p.kb <= 4) return launch_contig<DT, 4>(p, pool, st);
  if (p.kb <= 8) return launch_contig<DT, 8>(p, pool, st);
  return cudaErrorInvalidValue;
}

bool stage1_contig_supported(const Problem& p) { return p.layout == 1 && p.kb <= 8; }

cudaError_t run_stage1_contig(const Problem& p, uint64_t* pool, cudaStream_t st) {
  if (!stage1_contig_supported(p)) return cudaErrorNotSupported;
  switch (p.dtype) {
    case F32: return contig_t<F32>(p, pool, st);
    case BF16: return contig_t<BF16>(p, pool, st);
    case F16: return contig_t<F16>(p, pool, st);
  }
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------
template <int DT, int KB>
static cudaError_t launch_generic(const Problem& p, uint64_t* pool, cudaStream_t st) {
  dim3 grid((unsigned)((p.b + 255) / 256), (unsigned)std::min<int64_t>(p.m, 65535));
  s1_generic<DT, KB><<<grid, 256, 0, st>>>(p, pool);
  return cudaGetLastError();
}

template <int DT>
static cudaError_t generic_t(const Problem& p, uint64_t* pool, cudaStream_t st) {
  if (p.kb <= 1) return launch_generic<DT, 1>(p, pool, st);
  if (p.kb <= 2) return launch_generic<DT, 2>(p, pool, st);
  if (p.kb <= 4) return launch_generic<DT, 4>(p, pool, st);
  if (p.kb <= 8) return launch_generic<DT, 8>(p, pool, st);
  if (p.kb <= 16) return launch_generic<DT, 16>(p, pool, st);
  return cudaErrorInvalidValue;
}

cudaError_t run_stage1_generic(const Problem& p, uint64_t* pool, cudaStream_t st) {
  switch (p.dtype) {
    case F32: return generic_t<F32>(p, pool, st);
    case BF16: return generic_t<BF16>(p, pool, st);
    case F16: return generic_t<F16>(p, pool, st);
  }
  return cudaErrorInvalidValue;
}

static unsigned grid_for(int64_t total) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 64));
}

cudaError_t run_stage1_emit(const Problem& p, const uint64_t* pool, int64_t C, void* out_vals,
                            int64_t* out_idx, cudaStream_t st) {
  const unsigned g = grid_for(p.m * p.b * p.kb);
  switch (p.dtype) {
    case F32: s1_emit<F32><<<g, 256, 0, st>>>(p, pool, C, out_vals, out_idx); break;
    case BF16: s1_emit<BF16><<<g, 256, 0, st>>>(p, pool, C, out_vals, out_idx); break;
    case F16: s1_emit<F16><<<g, 256, 0, st>>>(p, pool, C, out_vals, out_idx); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace btk
