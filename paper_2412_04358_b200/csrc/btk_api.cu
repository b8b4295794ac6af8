// C ABI entry points (include/btk.h): validation, workspace planning and
// dispatch between the fused interleaved kernel and the generic path.
#include <cstring>

#include "../../include/btk.h"
#include "btk_internal.h"

using namespace btk;

namespace {

thread_local int g_last_cuda = 0;

int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return BTK_OK;
  g_last_cuda = (int)e;
  return BTK_ERR_CUDA;
}

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

size_t al(size_t v) { return (v + 255) & ~(size_t)255; }

bool dtype_ok(int d) { return d == BTK_F32 || d == BTK_BF16 || d == BTK_F16 || d == BTK_F64; }

int vbytes(int d) { return d == BTK_F64 ? 8 : (d == BTK_F32 ? 4 : 2); }

CompGeo geo_for(int dtype, int64_t space) {
  switch (dtype) {
    case BTK_F32: return make_geo<F32>(space);
    case BTK_BF16: return make_geo<BF16>(space);
    default: return make_geo<F16>(space);
  }
}

// Workspace carve-up of the generic path.
struct Plan {
  size_t pool = 0, mat = 0, s1a = 0, s1b = 0, s2a = 0, s2b = 0;
  size_t total() const { return al(pool) + al(mat) + al(s1a) + al(s1b) + al(s2a) + al(s2b); }
};

Plan plan_generic(int64_t m, int64_t n, int64_t k, int64_t b, int64_t kb) {
  Plan pl;
  (void)n;
  if (b == 1) {
    // whole-row exact select: only the k selected keys are stored (never
    // the row's n keys), then K2 sorts them
    pl.pool = (size_t)(m * k * 8);
    if (k > K2_SMALL_CAP) pl.s2a = pl.s2b = (size_t)(m * k * 8);
    return pl;
  }
  pl.pool = (size_t)(m * b * kb * 8);
  if (b * kb > K2_SMALL_CAP) pl.s2a = pl.s2b = (size_t)(m * k * 8);
  return pl;
}

// Workspace of btk_stage1: the pool, plus the in-place per-bucket sort's
// scratch when k_b > 16 exceeds one CTA's shared memory.
Plan plan_stage1(int64_t m, int64_t b, int64_t kb) {
  Plan pl;
  pl.pool = (size_t)(m * b * kb * 8);
  if (kb > 16 && kb > K2_SMALL_CAP) pl.s1a = pl.s1b = (size_t)(m * b * kb * 8);
  return pl;
}

// The plan of one call: the chunked Stage 2 (btk_pool.cu) when the pool is
// large and the vectorised Stage 1 applies, else plan_generic.
Plan plan_for(const Problem& p) {
  if (p.b > 1 && pool_chunked_ok(p)) {
    Plan pl;
    pl.pool = (size_t)(p.m * p.b * p.kb * 8);
    pl.s2a = pool_chunked_bytes(p);  // hist | tab | chunk buffer (fallback scratch aliases it + the pool)
    return pl;
  }
  return plan_generic(p.m, p.n, p.k, p.b, p.kb);
}

struct Carve {
  uint8_t* p;
  uint64_t* take(size_t bytes) {
    if (!bytes) return nullptr;
    uint64_t* r = reinterpret_cast<uint64_t*>(p);
    p += al(bytes);
    return r;
  }
};

// Stage 1 into the bucket-major pool (m x b*kb comps).  `sorted`: every
// bucket's k_b keys in canonical order (the stage1 API); Stage 2 only needs
// the set.
int stage1_pool(const Problem& p, const Plan& pl, Carve& cv, uint64_t* pool, cudaStream_t st, bool sorted) {
  if (p.b > 1 && stage1_vec_supported(p)) return cuda_status(run_stage1_vec(p, pool, st));
  if (stage1_contig_supported(p)) return cuda_status(run_stage1_contig(p, pool, st));
  if (p.kb <= 16) return cuda_status(run_stage1_generic(p, pool, st));
  // k_b > 16: exact per-bucket radix select straight from the scores (no
  // materialisation of the buckets), then, if asked, an in-place sort
  int rc = cuda_status(run_select_raw(p.dtype, p.x, p.row_stride, p.m, p.n, p.b, p.layout, p.kb, pool,
                                      p.geo, p.flag, st));
  if (rc || !sorted) return rc;
  K2Args a{};
  a.in = pool; a.in_stride = p.kb; a.nseg = p.m * p.b; a.L = p.kb; a.kk = p.kb;
  a.out_keys = pool; a.out_stride = p.kb; a.geo = p.geo;
  a.scratch_a = cv.take(pl.s1a);
  a.scratch_b = cv.take(pl.s1b);
  return cuda_status(run_k2(p.dtype, false, a, st));
}

int check_common(const void* x, int dtype, int layout, int64_t n, int64_t row_stride) {
  if (!dtype_ok(dtype)) return BTK_ERR_DTYPE;
  if (layout != BTK_INTERLEAVED && layout != BTK_CONTIGUOUS) return BTK_ERR_ASSIGNMENT;
  if (n >= (int64_t(1) << 31)) return BTK_ERR_SHAPE;
  if (row_stride < n) return BTK_ERR_SHAPE;
  if (x == nullptr) return BTK_ERR_SHAPE;
  if ((reinterpret_cast<uintptr_t>(x) % vbytes(dtype)) != 0) return BTK_ERR_ALIGNMENT;
  return BTK_OK;
}

}  // namespace

extern "C" {

int btk_validate(int64_t m, int64_t n, int64_t k, int64_t b, int64_t kb) {
  if (m < 1 || n < 1 || k < 1 || b < 1 || kb < 1) return BTK_ERR_NONPOSITIVE;
  if (k > n) return BTK_ERR_K_GT_N;
  if (b > n) return BTK_ERR_B_GT_N;
  if (kb > std::min<int64_t>(k, ceil_div(n, b))) return BTK_ERR_KB_RANGE;
  if (b * kb < k) return BTK_ERR_UNDERSAMPLED;
  return BTK_OK;
}

int btk_stage1_validate(int64_t n, int64_t b, int64_t kb) {
  if (n < 1) return BTK_ERR_SHAPE;
  if (b < 1 || b > n) return BTK_ERR_B_GT_N;
  if (kb < 1 || kb > ceil_div(n, b)) return BTK_ERR_KB_RANGE;
  return BTK_OK;
}

int64_t btk_stage1_count(int64_t n, int64_t b, int64_t kb, int layout) {
  if (btk_stage1_validate(n, b, kb) != BTK_OK) return -1;
  const int64_t q = n / b, r = n % b;
  if (kb <= q) return b * kb;
  (void)layout;  // both layouts have r buckets of q+1 and b-r of q
  return r * std::min<int64_t>(kb, q + 1) + (b - r) * std::min<int64_t>(kb, q);
}

size_t btk_workspace_bytes(int64_t m, int64_t n, int64_t k, int64_t b, int64_t kb, int dtype,
                           int layout) {
  if (btk_validate(m, n, k, b, kb) != BTK_OK || !dtype_ok(dtype)) return 0;
  if (dtype == BTK_F64) return f64_workspace_bytes(m, n, k, b, kb);
  // the fused plan depends on alignment only through x / row_stride; size it
  // for the aligned, contiguous case (the generic plan covers the rest)
  Problem p{};
  p.x = reinterpret_cast<const void*>(uintptr_t(256));
  p.row_stride = n;
  p.dtype = dtype;
  p.m = m; p.n = n; p.k = k; p.b = b; p.kb = kb;
  p.layout = layout;
  p.geo = geo_for(dtype, n);
  return std::max({plan_generic(m, n, k, b, kb).total(), plan_for(p).total(), fused_workspace_bytes(p),
                   xchg_supported(p) ? xchg_workspace_bytes(p) : (size_t)0});
}

size_t btk_plan_workspace_bytes(const void* x, int64_t row_stride, int dtype, int64_t m, int64_t n,
                                int64_t k, int64_t b, int64_t kb, int layout) {
  if (btk_validate(m, n, k, b, kb) != BTK_OK || !dtype_ok(dtype)) return 0;
  if (dtype == BTK_F64) return f64_workspace_bytes(m, n, k, b, kb);
  Problem p{};
  p.x = x;
  p.row_stride = row_stride;
  p.dtype = dtype;
  p.m = m; p.n = n; p.k = k; p.b = b; p.kb = kb;
  p.layout = layout;
  p.geo = geo_for(dtype, n);
  if (xchg_supported(p)) return xchg_workspace_bytes(p);
  if (fused_supported(p)) return fused_workspace_bytes(p);
  return plan_for(p).total();
}

int btk_uses_fused_path(int64_t m, int64_t n, int64_t k, int64_t b, int64_t kb, int dtype,
                        int layout, int64_t row_stride) {
  if (btk_validate(m, n, k, b, kb) != BTK_OK || !dtype_ok(dtype) || dtype == BTK_F64) return 0;
  Problem p{};
  p.x = reinterpret_cast<const void*>(uintptr_t(256));
  p.row_stride = row_stride;
  p.dtype = dtype;
  p.m = m; p.n = n; p.k = k; p.b = b; p.kb = kb;
  p.layout = layout;
  p.geo = geo_for(dtype, n);
  return (xchg_supported(p) || fused_supported(p)) ? 1 : 0;
}

int btk_kernel_family(int64_t m, int64_t n, int64_t k, int64_t b, int64_t kb, int dtype,
                      int layout, int64_t row_stride) {
  if (btk_validate(m, n, k, b, kb) != BTK_OK || !dtype_ok(dtype)) return -1;
  if (dtype == BTK_F64) return BTK_FAM_F64;
  Problem p{};
  p.x = reinterpret_cast<const void*>(uintptr_t(256));
  p.row_stride = row_stride;
  p.dtype = dtype;
  p.m = m; p.n = n; p.k = k; p.b = b; p.kb = kb;
  p.layout = layout;
  p.geo = geo_for(dtype, n);
  if (xchg_supported(p)) return BTK_FAM_XCHG;
  const int fk = fused_kind(p);
  if (fk) return fk;  // BTK_FAM_NARROW / WIDE / ROWS
  if (b == 1 || kb > 16) return BTK_FAM_MATERIALIZE;
  if (stage1_contig_supported(p)) return BTK_FAM_CONTIG;
  if (pool_chunked_ok(p)) return BTK_FAM_POOL_CHUNKED;
  return stage1_vec_supported(p) ? BTK_FAM_VEC_POOL : BTK_FAM_GENERIC;
}

int btk_launch_count(int64_t m, int64_t n, int64_t k, int64_t b, int64_t kb, int dtype,
                     int layout, int64_t row_stride) {
  if (btk_validate(m, n, k, b, kb) != BTK_OK || !dtype_ok(dtype)) return 0;
  if (dtype != BTK_F64) {
    Problem p{};
    p.x = reinterpret_cast<const void*>(uintptr_t(256));
    p.row_stride = row_stride; p.dtype = dtype;
    p.m = m; p.n = n; p.k = k; p.b = b; p.kb = kb; p.layout = layout; p.geo = geo_for(dtype, n);
    // the exchange pipeline + the persistent fallback kernel (exits at once
    // without overflow rows)
    if (xchg_supported(p)) return xchg_launch_count(p);
  }
  if (btk_uses_fused_path(m, n, k, b, kb, dtype, layout, row_stride)) return 1;
  if (dtype == BTK_F64) {
    auto segn = [](int64_t L, int64_t kk) { return L <= 8192 ? 1 : (kk <= 8192 ? 2 : 2); };
    if (b == 1) return segn(n, k);
    return (kb <= 16 ? 1 : segn(ceil_div(n, b), kb)) + segn(b * kb, k);
  }
  {
    Problem p{};
    p.x = reinterpret_cast<const void*>(uintptr_t(256));
    p.row_stride = row_stride; p.dtype = dtype;
    p.m = m; p.n = n; p.k = k; p.b = b; p.kb = kb; p.layout = layout; p.geo = geo_for(dtype, n);
    // s1_vec + pool_scatter + pool_sort + fallback (select/compact, sort); the memset is not a kernel
    if (b > 1 && pool_chunked_ok(p)) return 3 + (k <= K2_SMALL_CAP ? 2 : 2);
  }
  auto k2n = [](int64_t L, int64_t kk) { return L <= K2_SMALL_CAP ? 1 : 2; };
  if (b == 1) return 1 + k2n(k, k);  // raw select + sort of the k selected
  return 1 + k2n(b * kb, k);         // stage 1 (any form) + stage 2
}

int btk_approx_topk(const void* x, int64_t row_stride, int dtype, int64_t m, int64_t n, int64_t k,
                    int64_t b, int64_t kb, int layout, void* out_vals, int64_t* out_idx, void* ws,
                    size_t ws_bytes, uint32_t* flag, void* stream) {
  return btk_approx_topk_flags(x, row_stride, dtype, m, n, k, b, kb, layout, out_vals, out_idx, ws,
                               ws_bytes, flag, 0u, stream);
}

int btk_approx_topk_flags(const void* x, int64_t row_stride, int dtype, int64_t m, int64_t n, int64_t k,
                          int64_t b, int64_t kb, int layout, void* out_vals, int64_t* out_idx, void* ws,
                          size_t ws_bytes, uint32_t* flag, uint32_t flags, void* stream) {
  int rc = btk_validate(m, n, k, b, kb);
  if (rc) return rc;
  rc = check_common(x, dtype, layout, n, row_stride);
  if (rc) return rc;
  if (!out_vals || !out_idx) return BTK_ERR_SHAPE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == BTK_F64) {
    const size_t need = f64_workspace_bytes(m, n, k, b, kb);
    if (ws_bytes < need || (need && (reinterpret_cast<uintptr_t>(ws) & 255))) return BTK_ERR_WORKSPACE;
    return cuda_status(f64_approx_topk(x, row_stride, m, n, k, b, kb, layout, out_vals, out_idx, ws, flag, st));
  }
  Problem p{};
  p.x = x;
  p.row_stride = row_stride;
  p.dtype = dtype;
  p.m = m; p.n = n; p.k = k; p.b = b; p.kb = kb;
  p.layout = layout;
  p.geo = geo_for(dtype, n);
  p.flag = flag;
  p.flags = flags & BTK_INPUT_READY;
  if (xchg_supported(p)) {
    const size_t need = xchg_workspace_bytes(p);
    if (ws_bytes < need || (reinterpret_cast<uintptr_t>(ws) & 255)) return BTK_ERR_WORKSPACE;
    return cuda_status(run_xchg(p, ws, out_vals, out_idx, st));
  }
  if (fused_supported(p)) {
    const size_t need = fused_workspace_bytes(p);
    if (ws_bytes < need || (need && (reinterpret_cast<uintptr_t>(ws) & 255))) return BTK_ERR_WORKSPACE;
    return cuda_status(run_fused(p, out_vals, out_idx, ws, ws_bytes, st));
  }

  const Plan pl = plan_for(p);
  if (ws_bytes < pl.total() || (pl.total() && (reinterpret_cast<uintptr_t>(ws) & 255)))
    return BTK_ERR_WORKSPACE;
  Carve cv{static_cast<uint8_t*>(ws)};
  if (b > 1 && pool_chunked_ok(p)) {
    uint64_t* pool = cv.take(pl.pool);
    return cuda_status(run_pool_chunked(p, pool, cv.p, out_vals, out_idx, st));
  }
  if (b == 1) {
    // single bucket: the exact canonical top-k of the row — radix select of
    // the k largest straight from the scores, then K2 sorts those k
    uint64_t* sel = cv.take(pl.pool);
    uint64_t* s2a = cv.take(pl.s2a);
    uint64_t* s2b = cv.take(pl.s2b);
    rc = cuda_status(run_select_raw(dtype, x, row_stride, m, n, 1, layout, k, sel, p.geo, flag, st));
    if (rc) return rc;
    K2Args a{};
    a.in = sel; a.in_stride = k; a.nseg = m; a.L = k; a.kk = k;
    a.out_vals = out_vals; a.out_idx = out_idx; a.out_stride = k;
    a.geo = p.geo; a.scratch_a = s2a; a.scratch_b = s2b;
    return cuda_status(run_k2(dtype, true, a, st));
  }
  uint64_t* pool = cv.take(pl.pool);
  rc = stage1_pool(p, pl, cv, pool, st, false);
  if (rc) return rc;
  uint64_t* s2a = cv.take(pl.s2a);
  uint64_t* s2b = cv.take(pl.s2b);
  K2Args a{};
  a.in = pool; a.in_stride = b * kb; a.nseg = m; a.L = b * kb; a.kk = k;
  a.out_vals = out_vals; a.out_idx = out_idx; a.out_stride = k;
  a.geo = p.geo; a.scratch_a = s2a; a.scratch_b = s2b;
  return cuda_status(run_k2(dtype, true, a, st));
}

size_t btk_stage1_workspace_bytes(int64_t m, int64_t n, int64_t b, int64_t kb, int dtype,
                                  int layout) {
  (void)layout;
  if (btk_stage1_validate(n, b, kb) != BTK_OK || m < 1) return 0;
  if (dtype == BTK_F64) return f64_stage1_workspace_bytes(m, n, b, kb);
  return plan_stage1(m, b, kb).total();
}

int btk_stage1(const void* x, int64_t row_stride, int dtype, int64_t m, int64_t n, int64_t b,
               int64_t kb, int layout, void* out_vals, int64_t* out_idx, void* ws,
               size_t ws_bytes, uint32_t* flag, void* stream) {
  if (m < 1) return BTK_ERR_SHAPE;
  int rc = btk_stage1_validate(n, b, kb);
  if (rc) return rc;
  rc = check_common(x, dtype, layout, n, row_stride);
  if (rc) return rc;
  const size_t need = btk_stage1_workspace_bytes(m, n, b, kb, dtype, layout);
  if (ws_bytes < need || (need && (reinterpret_cast<uintptr_t>(ws) & 255))) return BTK_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == BTK_F64)
    return cuda_status(f64_stage1(x, row_stride, m, n, b, kb, layout, btk_stage1_count(n, b, kb, layout),
                                  out_vals, out_idx, ws, flag, st));
  Problem p{};
  p.x = x; p.row_stride = row_stride; p.dtype = dtype;
  p.m = m; p.n = n; p.k = std::min<int64_t>(n, b * kb); p.b = b; p.kb = kb;
  p.layout = layout; p.geo = geo_for(dtype, n); p.flag = flag;
  const Plan pl = plan_stage1(m, b, kb);
  Carve cv{static_cast<uint8_t*>(ws)};
  uint64_t* pool = cv.take(pl.pool);
  rc = stage1_pool(p, pl, cv, pool, st, true);
  if (rc) return rc;
  const int64_t C = btk_stage1_count(n, b, kb, layout);
  return cuda_status(run_stage1_emit(p, pool, C, out_vals, out_idx, st));
}

size_t btk_exact_workspace_bytes(int64_t m, int64_t n, int64_t k, int dtype) {
  return btk_workspace_bytes(m, n, k, 1, k, dtype, BTK_INTERLEAVED);
}

int btk_exact_topk(const void* x, int64_t row_stride, int dtype, int64_t m, int64_t n, int64_t k,
                   void* out_vals, int64_t* out_idx, void* ws, size_t ws_bytes, uint32_t* flag,
                   void* stream) {
  return btk_approx_topk(x, row_stride, dtype, m, n, k, 1, k, BTK_INTERLEAVED, out_vals, out_idx,
                         ws, ws_bytes, flag, stream);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// topk_with_indices: comps from (value, carried label)
namespace {
template <int DT>
__global__ void label_comps(const void* __restrict__ vals, const int64_t* __restrict__ labels,
                            int64_t total, uint64_t* __restrict__ out, CompGeo g, uint32_t* flag) {
  bool bad = false, badlab = false;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t bits = load_bits<DT>(vals, t);
    const int64_t lab = labels[t];
    bad |= nonfinite<DT>(bits);
    badlab |= (lab < 0) || (lab > (int64_t)g.imax);
    out[t] = make_comp(vkey<DT>(bits), (uint32_t)lab, is_negzero<DT>(bits), g);
  }
  const int b1 = __syncthreads_or(bad), b2 = __syncthreads_or(badlab);
  if (threadIdx.x == 0 && flag && (b1 || b2)) atomicOr(flag, (b1 ? 1u : 0u) | (b2 ? 2u : 0u));
}

__global__ void label_range(const int64_t* __restrict__ labels, int64_t total, uint32_t* flag) {
  bool bad = false;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lab = labels[t];
    bad |= (lab < 0) || (lab > 0x7FFFFFFF);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0 && flag) atomicOr(flag, 2u);
}

cudaError_t label_check(const int64_t* labels, int64_t total, uint32_t* flag, cudaStream_t st) {
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 16));
  label_range<<<grid, 256, 0, st>>>(labels, total, flag);
  return cudaGetLastError();
}
}  // namespace

extern "C" {

size_t btk_topk_with_indices_workspace_bytes(int64_t m, int64_t c, int64_t k, int dtype) {
  if (m < 1 || c < 1 || k < 1 || k > c) return 0;
  if (dtype == BTK_F64) return f64_pairs_workspace_bytes(m, c, k);
  size_t v = al((size_t)(m * c * 8));
  if (c > K2_SMALL_CAP) v += 2 * al((size_t)(m * k * 8));
  return v;
}

int btk_topk_with_indices(const void* values, const int64_t* labels, int dtype, int64_t m,
                          int64_t c, int64_t k, void* out_vals, int64_t* out_idx, void* ws,
                          size_t ws_bytes, uint32_t* flag, void* stream) {
  if (!dtype_ok(dtype)) return BTK_ERR_DTYPE;
  if (m < 1 || c < 1) return BTK_ERR_SHAPE;
  if (k < 1) return BTK_ERR_NONPOSITIVE;
  if (k > c) return BTK_ERR_K_GT_N;
  const size_t need = btk_topk_with_indices_workspace_bytes(m, c, k, dtype);
  if (ws_bytes < need || (reinterpret_cast<uintptr_t>(ws) & 255)) return BTK_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == BTK_F64) {
    if (c >= (int64_t(1) << 32)) return BTK_ERR_SHAPE;
    int rc = cuda_status(label_check(labels, m * c, flag, st));
    if (rc) return rc;
    return cuda_status(f64_topk_with_indices(values, labels, m, c, k, out_vals, out_idx, ws, flag, st));
  }
  const CompGeo g = geo_for(dtype, int64_t(1) << 31);
  Carve cv{static_cast<uint8_t*>(ws)};
  uint64_t* comps = cv.take((size_t)(m * c * 8));
  uint64_t* sa = c > K2_SMALL_CAP ? cv.take((size_t)(m * k * 8)) : nullptr;
  uint64_t* sb = c > K2_SMALL_CAP ? cv.take((size_t)(m * k * 8)) : nullptr;
  const int64_t total = m * c;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 64));
  switch (dtype) {
    case BTK_F32: label_comps<F32><<<grid, 256, 0, st>>>(values, labels, total, comps, g, flag); break;
    case BTK_BF16: label_comps<BF16><<<grid, 256, 0, st>>>(values, labels, total, comps, g, flag); break;
    default: label_comps<F16><<<grid, 256, 0, st>>>(values, labels, total, comps, g, flag); break;
  }
  int rc = cuda_status(cudaGetLastError());
  if (rc) return rc;
  K2Args a{};
  a.in = comps; a.in_stride = c; a.nseg = m; a.L = c; a.kk = k;
  a.out_vals = out_vals; a.out_idx = out_idx; a.out_stride = k;
  a.geo = g; a.scratch_a = sa; a.scratch_b = sb;
  a.unique = false;  // carried labels may repeat
  return cuda_status(run_k2(dtype, true, a, st));
}

int64_t btk_min_bytes(int64_t m, int64_t n, int64_t k, int64_t vb, int64_t ib) {
  return m * (n * vb + k * (vb + ib));
}

const char* btk_error_code(int s) {
  switch (s) {
    case BTK_OK: return "";
    case BTK_ERR_NONPOSITIVE: return "nonpositive";
    case BTK_ERR_K_GT_N: return "k_gt_n";
    case BTK_ERR_B_GT_N: return "b_gt_n";
    case BTK_ERR_KB_RANGE: return "kb_range";
    case BTK_ERR_UNDERSAMPLED: return "undersampled";
    case BTK_ERR_INSUFFICIENT_CANDIDATES: return "insufficient_candidates";
    case BTK_ERR_CHUNKS_RANGE: return "chunks_range";
    case BTK_ERR_ASSIGNMENT: return "assignment";
    case BTK_ERR_DTYPE: return "dtype";
    case BTK_ERR_SHAPE: return "shape";
    case BTK_ERR_WORKSPACE: return "workspace";
    case BTK_ERR_ALIGNMENT: return "alignment";
    case BTK_ERR_CUDA: return "cuda";
    case BTK_ERR_LABEL_RANGE: return "label_range";
  }
  return "unknown";
}

const char* btk_error_string(int s) {
  switch (s) {
    case BTK_OK: return "ok";
    case BTK_ERR_NONPOSITIVE: return "all of m, n, k, b, k_b must be positive integers";
    case BTK_ERR_K_GT_N: return "k > n";
    case BTK_ERR_B_GT_N: return "b > n";
    case BTK_ERR_KB_RANGE: return "k_b out of range 1..min(k, ceil(n/b))";
    case BTK_ERR_UNDERSAMPLED: return "b*kb < k";
    case BTK_ERR_INSUFFICIENT_CANDIDATES: return "stage 1 yields fewer than k candidates";
    case BTK_ERR_CHUNKS_RANGE: return "chunks_per_bucket must be >= 2";
    case BTK_ERR_ASSIGNMENT: return "unknown assignment";
    case BTK_ERR_DTYPE: return "unsupported dtype (float32, bfloat16, float16, float64)";
    case BTK_ERR_SHAPE: return "scores must be a non-empty m x n matrix";
    case BTK_ERR_WORKSPACE: return "workspace too small or not 256-byte aligned";
    case BTK_ERR_ALIGNMENT: return "misaligned device pointer";
    case BTK_ERR_CUDA: return "CUDA launch failed";
    case BTK_ERR_LABEL_RANGE: return "carried label outside [0, 2^31-1]";
  }
  return "unknown status";
}

int btk_last_cuda_error(void) { return g_last_cuda; }

const char* btk_version(void) { return "btk 0.1 sm_100a"; }

}  // extern "C"
