// Fused interleaved fast path: planning, dispatch and the internal entry
// points (btk_internal.h).  Kernels: btk_fused_impl.cuh; their per-dtype
// instantiations: btk_fused_{f32,bf16,f16}.cu.
#include "btk_fused_impl.cuh"

namespace btk {
namespace fz {
extern template cudaError_t launch_kb<F32>(const Plan&, int64_t, cudaStream_t);
extern template cudaError_t launch_kb<BF16>(const Plan&, int64_t, cudaStream_t);
extern template cudaError_t launch_kb<F16>(const Plan&, int64_t, cudaStream_t);
}  // namespace fz
using namespace fz;

bool fused_supported(const Problem& p) {
  Plan pl;
  return make_plan(p, pl);
}

int fused_kind(const Problem& p) {
  Plan pl;
  return make_plan(p, pl) ? (int)pl.kind : 0;
}

bool stage1_vec_supported(const Problem& p) {
  const int V = vec_of(p.dtype), esz = esz_of(p.dtype);
  if (p.layout != 0 || p.kb != kb_tmpl(p.kb) || V * p.kb > 16) return false;
  if (p.b % V || p.n % V) return false;
  if ((reinterpret_cast<uintptr_t>(p.x) & 15) || ((p.row_stride * esz) & 15)) return false;
  const int64_t s = (p.n + p.b - 1) / p.b;
  return s < 0xFFFF && p.m <= 65535;
}

template <int DT, int KB>
static cudaError_t launch_s1_vec(const Problem& p, uint64_t* pool, uint32_t* hist, cudaStream_t st,
                                 const int* rowmask) {
  constexpr int V = Vec<DT>::V;
  const int64_t G = p.b / V, s = (p.n + p.b - 1) / p.b;
  const int last_vec = (int)((p.n - (s - 1) * p.b) / V);
  const int64_t ngrp = (G + 255) / 256;
  // histogram flushes are per CTA: let a CTA cover several column groups
  // when there are CTAs to spare (cfg5: 8 CTAs per row instead of 32)
  const int groups = (hist && p.m * ngrp >= 148 * 32) ? 4 : 1;
  dim3 grid((unsigned)((ngrp + groups - 1) / groups), (unsigned)p.m);
  if (hist) {
    if (s <= 16) s1_vec<DT, KB, 16, true><<<grid, 256, 0, st>>>(p.x, p.row_stride, p.n, p.b, s, G, last_vec, p.geo, pool, p.flag, hist, groups, rowmask);
    else s1_vec<DT, KB, 8, true><<<grid, 256, 0, st>>>(p.x, p.row_stride, p.n, p.b, s, G, last_vec, p.geo, pool, p.flag, hist, groups, rowmask);
  } else {
    if (s <= 16) s1_vec<DT, KB, 16, false><<<grid, 256, 0, st>>>(p.x, p.row_stride, p.n, p.b, s, G, last_vec, p.geo, pool, p.flag, nullptr, groups, rowmask);
    else s1_vec<DT, KB, 8, false><<<grid, 256, 0, st>>>(p.x, p.row_stride, p.n, p.b, s, G, last_vec, p.geo, pool, p.flag, nullptr, groups, rowmask);
  }
  return cudaGetLastError();
}

template <int DT>
static cudaError_t s1_vec_dt(const Problem& p, uint64_t* pool, uint32_t* hist, cudaStream_t st,
                             const int* rowmask) {
  switch (p.kb) {
    case 1: return launch_s1_vec<DT, 1>(p, pool, hist, st, rowmask);
    case 2: return launch_s1_vec<DT, 2>(p, pool, hist, st, rowmask);
    case 4: return launch_s1_vec<DT, 4>(p, pool, hist, st, rowmask);
  }
  if constexpr (Vec<DT>::V * 8 <= 16) return launch_s1_vec<DT, 8>(p, pool, hist, st, rowmask);
  return cudaErrorNotSupported;
}

cudaError_t run_stage1_vec(const Problem& p, uint64_t* pool, cudaStream_t st, uint32_t* hist,
                           const int* rowmask) {
  if (!stage1_vec_supported(p)) return cudaErrorNotSupported;
  switch (p.dtype) {
    case F32: return s1_vec_dt<F32>(p, pool, hist, st, rowmask);
    case BF16: return s1_vec_dt<BF16>(p, pool, hist, st, rowmask);
    case F16: return s1_vec_dt<F16>(p, pool, hist, st, rowmask);
  }
  return cudaErrorInvalidValue;
}

size_t fused_workspace_bytes(const Problem& p) {
  Plan pl;
  return make_plan(p, pl) ? pl.ws : 0;
}

cudaError_t run_fused(const Problem& p, void* out_vals, int64_t* out_idx, void* ws, size_t ws_bytes,
                      cudaStream_t st) {
  Plan pl;
  if (!make_plan(p, pl)) return cudaErrorNotSupported;
  if (ws_bytes < pl.ws || (pl.ws && (reinterpret_cast<uintptr_t>(ws) & 255)))
    return cudaErrorInvalidValue;
  pl.na.out_vals = pl.wa.out_vals = pl.ra.out_vals = out_vals;
  pl.na.out_idx = pl.wa.out_idx = pl.ra.out_idx = out_idx;

  cudaError_t e = cudaErrorInvalidValue;
  switch (p.dtype) {
    case F32: e = launch_kb<F32>(pl, p.kb, st); break;
    case BF16: e = launch_kb<BF16>(pl, p.kb, st); break;
    case F16: e = launch_kb<F16>(pl, p.kb, st); break;
  }
  if (e != cudaSuccess && env_int("BTK_DEBUG", 0))
    fprintf(stderr, "[btk] fused launch failed: %s kind=%d nt=%d smem=%zu S=%d NS=%d T=%d R=%d G=%d m=%lld\n",
            cudaGetErrorString(e), (int)pl.kind, pl.nt, pl.smem, pl.na.S, pl.na.NS, pl.na.T, pl.na.R,
            pl.na.G, (long long)p.m);
  return e;
}

}  // namespace btk
