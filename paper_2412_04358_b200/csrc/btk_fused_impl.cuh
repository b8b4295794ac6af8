// Fused interleaved kernels (implementation header).  Included by
// btk_fused.cu (planning / dispatch / C-level entry points) and by the
// per-dtype translation units btk_fused_{f32,bf16,f16}.cu, which each
// instantiate launch_kb<DT> — the kernel templates of one dtype — so the
// three compile in parallel.
// Fused interleaved fast path: Stage 1 + Stage 2 + canonical write, one
// launch, no HBM round trip for the candidates.
//
// Interleaved buckets are the COLUMNS of a row viewed as an (s, b) row-major
// matrix (reference approx.py:112-131: grid[j, t] = j + b*t), so the
// reference's strided "gather cube" (approx.py:134-139) is free here: a
// contiguous run of view-rows is a dense tile whose columns are buckets.
//
// Two kernels:
//
//  fused_narrow  (b < V*NT: many view-rows per bucket; cfg1, cfg3, cfg4)
//      A cluster of S CTAs owns one row; CTA c streams view-rows
//      [c*s/S, (c+1)*s/S) through a shared-memory ring filled by
//      cp.async.bulk (TMA bulk copies, mbarrier complete_tx), one elected
//      thread issuing, every thread consuming.  Thread (r, g) owns the V
//      buckets of vector column g and every R-th view-row of a stage; it
//      keeps a register queue of the top-KB (value, slot) per bucket.
//      The R phase-queues are merged in smem, the S CTA partials are merged
//      by the leader through DSMEM, then the leader sorts the b*k_b
//      survivors and writes the first k.
//
//  fused_wide    (b >= V*NT: few view-rows per bucket; cfg2)
//      One CTA per row; each thread owns whole vector columns and streams
//      all s view-rows of them with 128-bit LDGs; the survivors go straight
//      into the smem pool.
//
// Per-element work (both): strict ">" on the exact float value keeps the
// earliest slot on ties == the reference argmax "first maximum"
// (approx.py:151-162); -0.0 == +0.0 and subnormals compare exactly (no
// FTZ, built with -ftz=false).  Stage 2 sorts composite keys descending ==
// the reference's two stable argsorts (exact.py:130-139).
//
// Outside the envelope (contiguous layout, b or n not a multiple of V,
// misaligned rows, V*k_b > 32, pool > 16384, smem overflow) the generic
// path (btk_stage1.cu + btk_select.cu) runs instead.
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdio>
#include <cstdlib>

#include "btk_internal.h"
#include "btk_lsd.cuh"
#include "btk_rank.cuh"
#include "btk_sort.cuh"

namespace cg = cooperative_groups;

namespace btk {

// Development timeline trace (BTK_TRACE=1): per CTA, globaltimer at start,
// first stage landed, streaming done, merged, end, ranked, SM id.  Read
// with btk_trace_read(); never enabled in production runs.
static __device__ unsigned long long g_trace[8192][8];  // per translation unit

namespace fz {  // fused-kernel internals, shared by the per-dtype translation units

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr int WIDE_NT = 512;
constexpr int WIDE_U = 8;                  // 16-byte loads in flight per thread
constexpr int64_t FUSED_POOL_CAP = 16384;  // survivors sorted in smem
constexpr size_t SMEM_LIMIT = 225 * 1024;  // dynamic; leaves room for static smem
constexpr int MAX_STAGES = 8;
#ifndef ROWS_MINB
#define ROWS_MINB 2
#endif
constexpr int NUM_SMS = 148;

template <int DT> struct Vec;
template <> struct Vec<F32> { static constexpr int V = 4; };
template <> struct Vec<BF16> { static constexpr int V = 8; };
template <> struct Vec<F16> { static constexpr int V = 8; };

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}

// 1-D TMA bulk copy global -> this CTA's shared memory, completion on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Asynchronous 8-byte store into another CTA's shared memory (DSMEM) that
// completes `bytes` on that CTA's mbarrier (st.async ... complete_tx).
__device__ __forceinline__ void st_async_remote_u64(const void* local_dst, const uint64_t* local_bar,
                                                    int rank, uint64_t v) {
  uint32_t rdst, rbar;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst) : "r"(smem_u32(local_dst)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_u32(local_bar)), "r"(rank));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(rdst),
               "l"(v), "r"(rbar)
               : "memory");
}

__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Launch-order contract for global writes.  Normally a kernel waits for its
// predecessor before its first input read (the predecessor may have
// produced the input), so writes need nothing more.  With early reads
// (BTK_INPUT_READY: the caller guarantees the input is not written by the
// preceding work in the stream) the kernel streams its input while the
// predecessor drains and waits only here, before its first global write.
__device__ __forceinline__ void pdl_wait_writes(bool early) {
  if (early) pdl_wait();
}

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// ------------------------------------------------------------------ element helpers
template <int DT>
__device__ __forceinline__ void unpack(const uint4& v, float (&f)[Vec<DT>::V]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  if constexpr (DT == F32) {
#pragma unroll
    for (int i = 0; i < 4; ++i) f[i] = __uint_as_float(w[i]);
  } else if constexpr (DT == BF16) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __uint_as_float(w[i] << 16);
      f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      f[2 * i] = __half2float(__ushort_as_half((unsigned short)(w[i] & 0xFFFFu)));
      f[2 * i + 1] = __half2float(__ushort_as_half((unsigned short)(w[i] >> 16)));
    }
  }
}

// OR-accumulator whose bit 31 (fp32) / bits 15,31 (16-bit) flag an all-ones exponent.
template <int DT>
__device__ __forceinline__ uint32_t nonfinite_bits(const uint4& v) {
  constexpr uint32_t M = DT == F32 ? 0x7F800000u : (DT == BF16 ? 0x7F807F80u : 0x7C007C00u);
  constexpr uint32_t A = DT == F32 ? 0x00800000u : (DT == BF16 ? 0x00800080u : 0x04000400u);
  return ((v.x & M) + A) | ((v.y & M) + A) | ((v.z & M) + A) | ((v.w & M) + A);
}

template <int DT>
__device__ __forceinline__ bool nonfinite_hit(uint32_t acc) {
  return DT == F32 ? (acc & 0x80000000u) != 0 : (acc & 0x80008000u) != 0;
}

template <int DT>
__device__ __forceinline__ uint32_t float_bits_to_raw(float f) {
  const uint32_t u = __float_as_uint(f);
  if constexpr (DT == F32) return u;
  else if constexpr (DT == BF16) return u >> 16;
  else return (uint32_t)__half_as_ushort(__float2half_rn(f));  // exact: f came from a half
}

// Register queue of the KB best (value, slot) of one bucket, descending.
template <int KB>
struct Queue {
  float v[KB];
  int t[KB];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int i = 0; i < KB; ++i) { v[i] = -__int_as_float(0x7F800000); t[i] = -1; }
  }
  __device__ __forceinline__ void push(float f, int tt) {
    if constexpr (KB == 1) {
      const bool gt = f > v[0];
      v[0] = gt ? f : v[0];
      t[0] = gt ? tt : t[0];
    } else {
      if (f > v[KB - 1]) {
#pragma unroll
        for (int i = KB - 1; i > 0; --i) {
          const bool up = f > v[i - 1];
          const bool here = f > v[i];
          v[i] = up ? v[i - 1] : (here ? f : v[i]);
          t[i] = up ? t[i - 1] : (here ? tt : t[i]);
        }
        const bool top = f > v[0];
        v[0] = top ? f : v[0];
        t[0] = top ? tt : t[0];
      }
    }
  }
};

// Insert a composite key into a descending KB-queue of comps.
template <int KB>
__device__ __forceinline__ void comp_push(uint64_t (&best)[KB], uint64_t c) {
  if (c > best[KB - 1]) {
#pragma unroll
    for (int z = KB - 1; z > 0; --z) best[z] = (c > best[z - 1]) ? best[z - 1] : (c > best[z] ? c : best[z]);
    best[0] = c > best[0] ? c : best[0];
  }
}

template <int DT>
__device__ __forceinline__ uint64_t comp_of(float f, int t, int64_t col, int64_t b,
                                            const CompGeo& g) {
  if (t < 0) return 0ull;
  const uint32_t raw = float_bits_to_raw<DT>(f);
  return make_comp(vkey<DT>(raw), (uint32_t)(t * b + col), is_negzero<DT>(raw), g);
}

template <int DT>
__device__ __forceinline__ void emit_comp(uint64_t c, int64_t pos, const CompGeo& g,
                                          void* out_vals, int64_t* out_idx) {
  uint32_t bits;
  int64_t idx;
  decode_comp<DT>(c, g, bits, idx);
  store_bits<DT>(out_vals, pos, bits);
  out_idx[pos] = idx;
}

// Stage 2 of one row's pool: the P survivors (ITEMS == 0, P <= 64: rank by
// counting; else the bucketing/rank engine
// of btk_rank.cuh with ITEMS >= P/NT keys per thread), then the canonical
// write of the first k.  `aux` is the engine's shared-memory scratch
// (rank_aux_bytes).  ITEMS is exact per kernel instance so the register
// budget of small-pool kernels is not set by the largest pools.

template <int DT, int NT, int ITEMS>
__device__ __forceinline__ void stage2_emit(uint64_t* pool, uint8_t* aux, int64_t P, int64_t k,
                                            int lognb, int64_t row, const CompGeo& geo,
                                            void* out_vals, int64_t* out_idx, bool trace_on = false,
                                            bool early = false) {
  if constexpr (ITEMS == 0) {
    // P <= 64: every key counts the keys above it (broadcast smem reads;
    // composite keys are unique) and writes itself at that rank — no sort
    pdl_wait_writes(early);
    for (int p = threadIdx.x; p < (int)P; p += NT) {
      const uint64_t x = pool[p];
      if (!x) continue;  // empty slot
      int f = 0;
#pragma unroll 8
      for (int j = 0; j < (int)P; ++j) f += pool[j] > x ? 1 : 0;
      if (f < k) emit_comp<DT>(x, row * k + f, geo, out_vals, out_idx);
    }
    return;
  }
  else {
    const RankSmem S = rank_smem(pool, aux, P, k, lognb, NT);
    rank_select_sort<DT, NT, ITEMS>(S, (int)P, (int)k, lognb, geo.ib);
    if (trace_on && threadIdx.x == 0 && blockIdx.x < 8192) g_trace[blockIdx.x][5] = gtime();
    pdl_wait_writes(early);
    for (int64_t q = threadIdx.x; q < k; q += NT)
      emit_comp<DT>(rs_key(pool, S.inv[q]), row * k + q, geo, out_vals, out_idx);
  }
}

inline int vec_of(int dtype) { return dtype == F32 ? 4 : 8; }
inline int esz_of(int dtype) { return dtype == F32 ? 4 : 2; }
inline int kb_tmpl(int64_t kb) { return kb <= 1 ? 1 : kb <= 2 ? 2 : kb <= 4 ? 4 : 8; }
// Engine keys per thread, rounded up to the instantiated set {0, 2, 8, 32}.
inline int sort_items_for(int64_t P, int NT) {
  if (P <= 64) return 0;
  if (P <= 2 * (int64_t)NT) return 2;
  if (P <= 8 * (int64_t)NT) return 8;
  return 32;
}
// Stage-2 shared memory after the pool's P keys.
inline size_t stage2_bytes(int64_t P, int64_t k, int NT) {
  if (P <= 64) return 64 * 8;
  return ((size_t)P * 8 + 127) / 128 * 128 + rank_aux_bytes(NT, rank_lognb(P), k, P);
}
inline size_t a16(size_t v) { return (v + 127) & ~(size_t)127; }

// Tuning overrides for launch-shape sweeps (unset in production runs).
inline int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return (v && *v) ? std::atoi(v) : dflt;
}

// Programmatic dependent launch (griddepcontrol): on by default.  Kernels
// wait for their predecessor before the first read, so only the launch and
// prologue overlap the previous kernel's tail (cfg1 +1.8%); BTK_PDL=0
// disables it.
inline bool pdl_enabled() {
  static const int v = env_int("BTK_PDL", 1);
  return v != 0;
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(addr));
  return r;
}

// Per-thread stage-1 state for one vector column (V adjacent buckets).
// row(v, trel) consumes one 16-byte vector of view-row trel (relative to
// the CTA's first view-row); spill() writes KB composite keys per bucket.
// Non-finite detection folds into one FMA per element: x*0 + acc is NaN
// iff some x was NaN or +-inf.
template <int DT, int KB>
struct Scanner {
  static constexpr int V = Vec<DT>::V;
  Queue<KB> q[V];
  float nf[V];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int e = 0; e < V; ++e) { q[e].init(); nf[e] = 0.f; }
  }
  __device__ __forceinline__ void row(const uint4& v, int trel) {
    float f[V];
    unpack<DT>(v, f);
#pragma unroll
    for (int e = 0; e < V; ++e) {
      nf[e] = fmaf(f[e], 0.f, nf[e]);
      q[e].push(f[e], trel);
    }
  }
  __device__ __forceinline__ bool nonfinite() const {
    bool bad = false;
#pragma unroll
    for (int e = 0; e < V; ++e) bad |= (nf[e] != nf[e]);
    return bad;
  }
  template <int KBS>
  __device__ __forceinline__ void spill(uint64_t* dst, int g, int64_t b, int64_t t_begin,
                                        const CompGeo& geo) const {
    each_comp(g, b, t_begin, geo, [&](int64_t col, int z, uint64_t c) { dst[col * KBS + z] = c; });
  }
  // f(col, z, comp) for the KB survivors of each of the V buckets (0 = empty)
  template <class F>
  __device__ __forceinline__ void each_comp(int g, int64_t b, int64_t t_begin, const CompGeo& geo,
                                            F&& f) const {
#pragma unroll
    for (int e = 0; e < V; ++e) {
      const int64_t col = (int64_t)g * V + e;
#pragma unroll
      for (int z = 0; z < KB; ++z) {
        const int t = q[e].t[z] < 0 ? -1 : (int)(t_begin + q[e].t[z]);
        f(col, z, comp_of<DT>(q[e].v[z], t, col, b, geo));
      }
    }
  }
};

// k_b = 1 on 16-bit data: two buckets per 32-bit word, all packed.
// Per word: HSET2 mask (strict >), two LOP3 bit-selects (value bits kept
// exactly, so the sign of zero survives) and one HFMA2 for the finite check
// -> 2 instructions per element.  Slot codes are 16-bit offsets from the
// CTA's first view-row (planner guarantees < 0xFFFF rows per CTA).
template <int DT>
struct Scanner16x2 {
  static constexpr uint32_t NEG_INF2 = DT == BF16 ? 0xFF80FF80u : 0xFC00FC00u;
  uint32_t m2[4], c2[4], nf2[4];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int w = 0; w < 4; ++w) { m2[w] = NEG_INF2; c2[w] = 0xFFFFFFFFu; nf2[w] = 0u; }
  }
  __device__ __forceinline__ static uint32_t gt_mask(uint32_t x, uint32_t y) {
    if constexpr (DT == BF16) {
      return __hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&x),
                         *reinterpret_cast<const __nv_bfloat162*>(&y));
    } else {
      return __hgt2_mask(*reinterpret_cast<const __half2*>(&x), *reinterpret_cast<const __half2*>(&y));
    }
  }
  __device__ __forceinline__ static uint32_t fma0(uint32_t x, uint32_t acc) {
    if constexpr (DT == BF16) {
      __nv_bfloat162 r = __hfma2(*reinterpret_cast<const __nv_bfloat162*>(&x),
                                 __nv_bfloat162(__float2bfloat16(0.f), __float2bfloat16(0.f)),
                                 *reinterpret_cast<const __nv_bfloat162*>(&acc));
      return *reinterpret_cast<uint32_t*>(&r);
    } else {
      __half2 r = __hfma2(*reinterpret_cast<const __half2*>(&x), __half2(__float2half(0.f), __float2half(0.f)),
                          *reinterpret_cast<const __half2*>(&acc));
      return *reinterpret_cast<uint32_t*>(&r);
    }
  }
  __device__ __forceinline__ void row(const uint4& v, int trel) {
    const uint32_t code = (uint32_t)trel * 0x10001u;
    const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const uint32_t mask = gt_mask(w4[w], m2[w]);
      m2[w] = (w4[w] & mask) | (m2[w] & ~mask);
      c2[w] = (code & mask) | (c2[w] & ~mask);
      nf2[w] = fma0(w4[w], nf2[w]);
    }
  }
  __device__ __forceinline__ bool nonfinite() const {
    constexpr uint32_t E = DT == BF16 ? 0x7F80u : 0x7C00u;
    bool bad = false;
#pragma unroll
    for (int w = 0; w < 4; ++w)
      bad |= ((nf2[w] & 0x7FFFu) > E) || (((nf2[w] >> 16) & 0x7FFFu) > E);
    return bad;
  }
  template <int KBS>
  __device__ __forceinline__ void spill(uint64_t* dst, int g, int64_t b, int64_t t_begin,
                                        const CompGeo& geo) const {
    each_comp(g, b, t_begin, geo, [&](int64_t col, int, uint64_t c) {
      dst[col * KBS] = c;
#pragma unroll
      for (int z = 1; z < KBS; ++z) dst[col * KBS + z] = 0ull;
    });
  }
  template <class F>
  __device__ __forceinline__ void each_comp(int g, int64_t b, int64_t t_begin, const CompGeo& geo,
                                            F&& f) const {
#pragma unroll
    for (int w = 0; w < 4; ++w) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t col = (int64_t)g * 8 + 2 * w + h;
        const uint32_t raw = (m2[w] >> (16 * h)) & 0xFFFFu;
        const uint32_t code = (c2[w] >> (16 * h)) & 0xFFFFu;
        uint64_t c = 0ull;
        if (code != 0xFFFFu) {
          const int64_t idx = (t_begin + code) * b + col;
          c = make_comp(vkey<DT>(raw), (uint32_t)idx, is_negzero<DT>(raw), geo);
        }
        f(col, 0, c);
      }
    }
  }
  // f(i, raw, code) per survivor i = column offset in the group (code
  // 0xFFFF = empty): the 16-bit value and its view-row, no composite key
  template <class F>
  __device__ __forceinline__ void each_raw(F&& f) const {
#pragma unroll
    for (int w = 0; w < 4; ++w) {
#pragma unroll
      for (int h = 0; h < 2; ++h) f(2 * w + h, (m2[w] >> (16 * h)) & 0xFFFFu, (c2[w] >> (16 * h)) & 0xFFFFu);
    }
  }
};

template <> struct Scanner<BF16, 1> : Scanner16x2<BF16> {};
template <> struct Scanner<F16, 1> : Scanner16x2<F16> {};

// k_b = 2 on 16-bit data, packed like Scanner16x2: per 32-bit word two
// HSET2 masks (x > first, x > second) and bit-selects that shift the first
// into second place when x beats it -> ~4 instructions per element.  Ties
// keep the earlier slot (strict >), as the float Queue does.
template <int DT>
struct Scanner16x2K2 {
  using S1 = Scanner16x2<DT>;
  uint32_t m1[4], m2[4], c1[4], c2[4], nf2[4];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      m1[w] = m2[w] = S1::NEG_INF2;
      c1[w] = c2[w] = 0xFFFFFFFFu;
      nf2[w] = 0u;
    }
  }
  __device__ __forceinline__ void row(const uint4& v, int trel) {
    const uint32_t code = (uint32_t)trel * 0x10001u;
    const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const uint32_t x = w4[w];
      const uint32_t g1 = S1::gt_mask(x, m1[w]);
      const uint32_t g2 = S1::gt_mask(x, m2[w]);
      const uint32_t s2 = (x & g2) | (m2[w] & ~g2);
      const uint32_t t2 = (code & g2) | (c2[w] & ~g2);
      m2[w] = (m1[w] & g1) | (s2 & ~g1);
      c2[w] = (c1[w] & g1) | (t2 & ~g1);
      m1[w] = (x & g1) | (m1[w] & ~g1);
      c1[w] = (code & g1) | (c1[w] & ~g1);
      nf2[w] = S1::fma0(x, nf2[w]);
    }
  }
  __device__ __forceinline__ bool nonfinite() const {
    constexpr uint32_t E = DT == BF16 ? 0x7F80u : 0x7C00u;
    bool bad = false;
#pragma unroll
    for (int w = 0; w < 4; ++w)
      bad |= ((nf2[w] & 0x7FFFu) > E) || (((nf2[w] >> 16) & 0x7FFFu) > E);
    return bad;
  }
  template <int KBS>
  __device__ __forceinline__ void spill(uint64_t* dst, int g, int64_t b, int64_t t_begin,
                                        const CompGeo& geo) const {
    each_comp(g, b, t_begin, geo, [&](int64_t col, int z, uint64_t c) {
      dst[col * KBS + z] = c;
      if (z == 1) {
#pragma unroll
        for (int q = 2; q < KBS; ++q) dst[col * KBS + q] = 0ull;
      }
    });
  }
  template <class F>
  __device__ __forceinline__ void each_comp(int g, int64_t b, int64_t t_begin, const CompGeo& geo,
                                            F&& f) const {
#pragma unroll
    for (int w = 0; w < 4; ++w) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t col = (int64_t)g * 8 + 2 * w + h;
#pragma unroll
        for (int z = 0; z < 2; ++z) {
          const uint32_t raw = ((z ? m2[w] : m1[w]) >> (16 * h)) & 0xFFFFu;
          const uint32_t code = ((z ? c2[w] : c1[w]) >> (16 * h)) & 0xFFFFu;
          uint64_t c = 0ull;
          if (code != 0xFFFFu) {
            const int64_t idx = (t_begin + code) * b + col;
            c = make_comp(vkey<DT>(raw), (uint32_t)idx, is_negzero<DT>(raw), geo);
          }
          f(col, z, c);
        }
      }
    }
  }
  // f(i, raw, code) per survivor i = 2 * column offset + z (see Scanner16x2)
  template <class F>
  __device__ __forceinline__ void each_raw(F&& f) const {
#pragma unroll
    for (int w = 0; w < 4; ++w) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        f(2 * (2 * w + h), (m1[w] >> (16 * h)) & 0xFFFFu, (c1[w] >> (16 * h)) & 0xFFFFu);
        f(2 * (2 * w + h) + 1, (m2[w] >> (16 * h)) & 0xFFFFu, (c2[w] >> (16 * h)) & 0xFFFFu);
      }
    }
  }
};
template <> struct Scanner<BF16, 2> : Scanner16x2K2<BF16> {};
template <> struct Scanner<F16, 2> : Scanner16x2K2<F16> {};

// ============================================================ narrow (TMA ring, cluster)
struct NarrowArgs {
  const void* x;
  int64_t row_stride;  // elements
  int64_t m, n, k, b, kb, s;
  int G, R;            // vector columns, view-row phases per stage
  int S;               // CTAs per row (cluster size)
  int T;               // view-rows per ring stage
  int NS;              // ring stages
  int sort_items;
  int64_t P;
  int last_vec;        // valid vector columns of view-row s-1
  size_t stage_bytes;  // T * b * esz
  size_t scratch_off, part_off, pool_off, aux_off;  // post-scan layout (aliases the ring)
  int lognb;
  CompGeo geo;
  void* out_vals;
  int64_t* out_idx;
  uint32_t* flag;
  int trace;
  int early;  // read the input before the predecessor completes (BTK_INPUT_READY)
};

template <int KB>
__host__ __device__ constexpr int kb_store() { return KB; }

// Tail shared by the cluster kernels: fold the R phase queues, push the
// CTA's partial into the leader's slot (DSMEM store for crank > 0), one
// cluster barrier, then the leader merges the S slots and runs Stage 2.
template <int DT, int KB, int NT, int ITEMS>
__device__ __forceinline__ void narrow_tail(const NarrowArgs& a, uint8_t* smem, Scanner<DT, KB>& sc,
                                            bool active, int r, int g, int64_t t_begin,
                                            uint32_t bad, int64_t row, int crank, bool tr,
                                            cg::cluster_group& cluster, uint64_t* pbar) {
  const int tid = threadIdx.x;
  const int64_t b = a.b;
  const int R = a.R;
  uint64_t* scratch = reinterpret_cast<uint64_t*>(smem + a.scratch_off);
  uint64_t* part = reinterpret_cast<uint64_t*>(smem + a.part_off);
  uint64_t* pool = reinterpret_cast<uint64_t*>(smem + a.pool_off);
  if (active) sc.template spill<KB>(scratch + (int64_t)r * b * KB, g, b, t_begin, a.geo);
  __syncthreads();
  // fold the R phase queues; partners push their partial into the leader's
  // slot c with st.async (completing bytes on the leader's mbarrier) and are
  // done — no cluster barrier, no remote reads
  if (a.S > 1 && crank != 0) cluster_wait_acquire();  // leader's pbar initialised
  for (int64_t j = tid; j < b; j += NT) {
    uint64_t best[KB];
#pragma unroll
    for (int z = 0; z < KB; ++z) best[z] = 0ull;
    for (int rr = 0; rr < R; ++rr) {
#pragma unroll
      for (int z = 0; z < KB; ++z) comp_push<KB>(best, scratch[((int64_t)rr * b + j) * KB + z]);
    }
    if (crank == 0) {
#pragma unroll
      for (int z = 0; z < KB; ++z) part[j * KB + z] = best[z];
    } else {
#pragma unroll
      for (int z = 0; z < KB; ++z)
        st_async_remote_u64(part + ((int64_t)crank * b + j) * KB + z, pbar, 0, best[z]);
    }
  }
  const bool anybad = __syncthreads_or(bad);
  if (anybad && tid == 0 && a.flag) atomicOr(a.flag, 1u);
  if (a.S > 1 && crank == 0) {
    cluster_wait_acquire();
    mbar_wait(pbar, 0u);  // all partner partials landed
  }
  if (crank == 0) {
    for (int64_t j = tid; j < b; j += NT) {
      uint64_t best[KB];
#pragma unroll
      for (int z = 0; z < KB; ++z) best[z] = part[j * KB + z];
      for (int c = 1; c < a.S; ++c) {
#pragma unroll
        for (int z = 0; z < KB; ++z) comp_push<KB>(best, part[((int64_t)c * b + j) * KB + z]);
      }
#pragma unroll
      for (int z = 0; z < KB; ++z)
        if (z < a.kb) pool[j * a.kb + z] = best[z];
    }
  }
  if (tr) g_trace[blockIdx.x][3] = gtime();
  if (crank != 0) {
    if (tr) g_trace[blockIdx.x][4] = gtime();
    return;
  }
  __syncthreads();
  if (tr) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_trace[blockIdx.x][6] = smid;
  }
  stage2_emit<DT, NT, ITEMS>(pool, smem + a.aux_off, a.P, a.k, a.lognb, row, a.geo, a.out_vals,
                            a.out_idx, a.trace != 0, a.early != 0);
  if (tr) g_trace[blockIdx.x][4] = gtime();}

template <int DT, int KB, int NT, int ITEMS>
__global__ void __launch_bounds__(NT) fused_narrow(NarrowArgs a) {
  constexpr int V = Vec<DT>::V;
  constexpr int LB = (KB <= 2) ? 8 : 4;  // smem vectors in flight per thread
  constexpr int ESZ = VT<DT>::W / 8;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[MAX_STAGES];
  __shared__ __align__(8) uint64_t pbar;  // leader: partials of the partner CTAs

  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const bool tr = a.trace && threadIdx.x == 0 && blockIdx.x < 8192;
  if (tr) g_trace[blockIdx.x][0] = gtime();
  const int64_t row = blockIdx.x / a.S;
  const int tid = threadIdx.x;
  const int64_t b = a.b, s = a.s;
  const uint8_t* rowp = static_cast<const uint8_t*>(a.x) + row * a.row_stride * ESZ;
  const int64_t t_begin = (s * crank) / a.S, t_end = (s * (crank + 1)) / a.S;
  const int nstages = (int)((t_end - t_begin + a.T - 1) / a.T);

  if (tid == 0) {
    for (int i = 0; i < a.NS; ++i) mbar_init(&full[i], 1);
    if (a.S > 1 && crank == 0) {
      // the partners' partials land here by st.async (complete_tx)
      mbar_init(&pbar, 1);
      mbar_expect_tx(&pbar, (uint32_t)((a.S - 1) * a.b * kb_store<KB>() * 8));
    }
    fence_barrier_init();
  }
  // publish the leader's barrier cluster-wide; partners wait on this phase
  // only right before their first remote store (long since complete)
  if (a.S > 1) cluster_arrive_release();
  // Programmatic dependent launch: let the next launch in the stream get
  // resident during our tail, and wait for our predecessor to finish (its
  // writes may be our input) before the first read.
  pdl_trigger();
  if (!a.early) pdl_wait();
  __syncthreads();

  uint64_t policy = 0;
  auto issue = [&](int i) {
    const int slot = i % a.NS;
    const int64_t t0 = t_begin + (int64_t)i * a.T;
    const int64_t rows = min((int64_t)a.T, t_end - t0);
    int64_t elems = rows * b;
    if (t0 + rows == s) elems -= b - (int64_t)a.last_vec * V;  // ragged final view-row
    const uint32_t bytes = (uint32_t)(elems * ESZ);
    // order the consumers' generic-proxy reads of this slot before the
    // async-proxy (TMA) overwrite
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&full[slot], bytes);
    bulk_g2s(smem + (size_t)slot * a.stage_bytes, rowp + t0 * b * ESZ, bytes, &full[slot], policy);
  };
  if (tid == 0) {
    policy = evict_first_policy();
    const int pre = min(a.NS, nstages);
    for (int i = 0; i < pre; ++i) issue(i);
  }

  const int G = a.G, R = a.R;
  const int r = tid / G, g = tid - r * G;
  const bool active = r < R;
  Scanner<DT, KB> sc;
  sc.init();
  const uint32_t smem_base = smem_u32(smem) + (uint32_t)(g * V * ESZ);
  const uint32_t row_step = (uint32_t)(R * b * ESZ);

  for (int i = 0; i < nstages; ++i) {
    const int slot = i % a.NS;
    mbar_wait(&full[slot], (uint32_t)((i / a.NS) & 1));
    if (tr && i == 0) g_trace[blockIdx.x][1] = gtime();
    const int64_t t0 = t_begin + (int64_t)i * a.T;
    const int rows = (int)min((int64_t)a.T, t_end - t0);
    // the ragged final view-row (only partially valid) is handled last
    const bool ragged = (t0 + rows == s) && (a.last_vec < G);
    const int rows_main = rows - (ragged ? 1 : 0);
    if (active) {
      uint32_t addr = smem_base + (uint32_t)(slot * a.stage_bytes) + (uint32_t)(r * b * ESZ);
      const int trel0 = (int)(t0 - t_begin);
      // LB shared-memory loads issued back to back, then consumed: the scan
      // of a stage is issue/latency-bound once HBM delivers (cfg3: one CTA
      // per SM), so the loads must not wait on the previous row's compute
      int rr = r;
      for (; rr + (LB - 1) * R < rows_main; rr += LB * R) {
        uint4 v[LB];
#pragma unroll
        for (int u = 0; u < LB; ++u) v[u] = lds128(addr + (uint32_t)u * row_step);
#pragma unroll
        for (int u = 0; u < LB; ++u) sc.row(v[u], trel0 + rr + u * R);
        addr += (uint32_t)LB * row_step;
      }
      for (; rr < rows_main; rr += R) {
        sc.row(lds128(addr), trel0 + rr);
        addr += row_step;
      }
      if (ragged && (rows - 1) % R == r && g < a.last_vec)
        sc.row(lds128(smem_base + (uint32_t)(slot * a.stage_bytes) + (uint32_t)((rows - 1) * b * ESZ)),
               trel0 + rows - 1);
    }
    __syncthreads();  // slot consumed by every thread
    if (tid == 0 && i + a.NS < nstages) issue(i + a.NS);
  }
  const uint32_t bad = sc.nonfinite() ? 1u : 0u;
  if (tr) g_trace[blockIdx.x][2] = gtime();

  narrow_tail<DT, KB, NT, ITEMS>(a, smem, sc, active, r, g, t_begin, bad, row, crank, tr, cluster, &pbar);
}


// ============================================================ rows (one warp per row)
// Many short rows (cfg4: 4096 x 32768, b = 512): block-level barriers and
// a CTA-wide sort per row would serialise the tail of every row.  Here a
// WARP owns a row end to end: lane l streams vector columns l, l+32, ...
// (GPL per lane) with U 128-bit loads in flight per column, keeps the
// register queues, spills its b*k_b survivors to a per-warp shared pool,
// and runs a warp-synchronous version of the bucketing/rank engine
// (btk_rank.cuh) — only __syncwarp, so the 32 warps of an SM progress
// independently and one warp's tail overlaps the others' streaming.
struct RowsArgs {
  const void* x;
  int64_t row_stride;
  int64_t m, n, k, b, kb, s;
  int G, last_vec, lognb;
  int64_t P;
  size_t warp_smem, inv_off, hist_off, bid_off;
  CompGeo geo;
  void* out_vals;
  int64_t* out_idx;
  uint32_t* flag;
  int early;  // read the input before the predecessor completes (BTK_INPUT_READY)
};

template <int DT, int KB, int GPL, int U, int ITEMS>
__global__ void __launch_bounds__(256, ROWS_MINB) fused_rows(RowsArgs a) {
  constexpr int V = Vec<DT>::V;
  constexpr int ESZ = VT<DT>::W / 8;
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* wsm = smem + (size_t)warp * a.warp_smem;
  uint64_t* pool = reinterpret_cast<uint64_t*>(wsm);
  uint16_t* inv = reinterpret_cast<uint16_t*>(wsm + a.inv_off);
  uint32_t* hist = reinterpret_cast<uint32_t*>(wsm + a.hist_off);
  uint16_t* bid = reinterpret_cast<uint16_t*>(wsm + a.bid_off);
  const int64_t b = a.b, s = a.s;
  const int G = a.G;
  uint32_t bad = 0;
  pdl_trigger();
  if (!a.early) pdl_wait();
  for (int64_t row = (int64_t)blockIdx.x * 8 + warp; row < a.m; row += (int64_t)gridDim.x * 8) {
    const uint8_t* rowp = static_cast<const uint8_t*>(a.x) + row * a.row_stride * ESZ;
    Scanner<DT, KB> sc[GPL];
#pragma unroll
    for (int j = 0; j < GPL; ++j) sc[j].init();
    // all GPL columns' loads of U view-rows in flight together (GPL*U
    // 16-byte loads per lane); the ragged final view-row, if any, last
    const int64_t s_full = (a.last_vec < G) ? s - 1 : s;
    int64_t t0 = 0;
    for (; t0 + U <= s_full; t0 += U) {
      uint4 v[GPL][U];
#pragma unroll
      for (int j = 0; j < GPL; ++j) {
        const int g = lane + 32 * j;
#pragma unroll
        for (int u = 0; u < U; ++u)
          v[j][u] = (g < G) ? ldg_stream(rowp + ((t0 + u) * b + (int64_t)g * V) * ESZ) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int j = 0; j < GPL; ++j) {
        if (lane + 32 * j < G) {
#pragma unroll
          for (int u = 0; u < U; ++u) sc[j].row(v[j][u], (int)(t0 + u));
        }
      }
    }
#pragma unroll
    for (int j = 0; j < GPL; ++j) {
      const int g = lane + 32 * j;
      if (g < G) {
        const int64_t s_eff = (g < a.last_vec) ? s : s - 1;
        for (int64_t t = t0; t < s_eff; ++t)
          sc[j].row(ldg_stream(rowp + (t * b + (int64_t)g * V) * ESZ), (int)t);
      }
    }
#pragma unroll
    for (int j = 0; j < GPL; ++j) {
      const int g = lane + 32 * j;
      if (g < G) {
        bad |= sc[j].nonfinite() ? 1u : 0u;
        sc[j].template spill<KB>(pool, g, b, 0, a.geo);
      }
    }
    __syncwarp();
    warp_rank_sort<DT, ITEMS>(pool, (int)a.P, (int)a.k, inv, bid, hist, a.lognb, a.geo.ib);
    pdl_wait_writes(a.early != 0);
    for (int64_t q = lane; q < a.k; q += 32)
      emit_comp<DT>(rs_key(pool, inv[q]), row * a.k + q, a.geo, a.out_vals, a.out_idx);
    __syncwarp();
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0 && a.flag) atomicOr(a.flag, 1u);
}

// ============================================================ wide (LDG, one CTA per row)
struct WideArgs {
  const void* x;
  int64_t row_stride;
  int64_t m, n, k, b, kb, s, G;
  int sort_items;
  int64_t P;
  int last_vec;
  size_t pool_off, aux_off;
  int lognb;
  CompGeo geo;
  void* out_vals;
  int64_t* out_idx;
  uint32_t* flag;
  int trace;
  int early;  // read the input before the predecessor completes (BTK_INPUT_READY)
  int lsd_lowbit;  // > 0: large pool, stable LSD Stage 2 from this bit (btk_lsd.cuh)
};

template <int DT, int KB, int NT, int U, int ITEMS>
__global__ void __launch_bounds__(NT, 1) fused_wide(WideArgs a) {
  constexpr int V = Vec<DT>::V;
  constexpr int ESZ = VT<DT>::W / 8;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* pool = reinterpret_cast<uint64_t*>(smem + a.pool_off);
  const int64_t row = blockIdx.x;
  const uint8_t* rowp = static_cast<const uint8_t*>(a.x) + row * a.row_stride * ESZ;
  const int64_t b = a.b, s = a.s;
  const int tid = threadIdx.x;
  uint32_t bad = 0;
  pdl_trigger();
  if (!a.early) pdl_wait();
  const bool tr = a.trace && tid == 0 && blockIdx.x < 8192;
  if (tr) g_trace[blockIdx.x][0] = gtime();
  auto spill_col = [&](Queue<KB> (&q)[V], int64_t g) {
#pragma unroll
    for (int e = 0; e < V; ++e) {
      const int64_t col = g * V + e;
#pragma unroll
      for (int z = 0; z < KB; ++z) {
        if (z < a.kb) {
          const int p = (int)(col * a.kb + z);  // bucket-id order
          pool[a.lsd_lowbit ? lsd::pad32(p) : p] = comp_of<DT>(q[e].v[z], q[e].t[z], col, b, a.geo);
        }
      }
    }
  };
  if (s <= U) {
    // short columns (cfg2: s = 8): one load round per vector column, so
    // software-pipeline across columns — the next column's loads are in
    // flight while this one is scanned (2*s loads per thread)
    auto load_col = [&](uint4 (&v)[U], int64_t g) {
      const uint8_t* colp = rowp + g * V * ESZ;
      const int64_t s_eff = (g < a.last_vec) ? s : s - 1;  // ragged final view-row
#pragma unroll
      for (int u = 0; u < U; ++u)
        v[u] = (g < a.G && u < s_eff) ? ldg_stream(colp + (int64_t)u * b * ESZ) : make_uint4(0u, 0u, 0u, 0u);
    };
    uint4 cur[U], nxt[U];
    int64_t g = tid;
    load_col(cur, g);
    for (; g < a.G; g += NT) {
      load_col(nxt, g + NT);
      Queue<KB> q[V];
#pragma unroll
      for (int e = 0; e < V; ++e) q[e].init();
      const int64_t s_eff = (g < a.last_vec) ? s : s - 1;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (u < s_eff) {
          bad |= nonfinite_bits<DT>(cur[u]);
          float f[V];
          unpack<DT>(cur[u], f);
#pragma unroll
          for (int e = 0; e < V; ++e) q[e].push(f[e], u);
        }
      }
      spill_col(q, g);
#pragma unroll
      for (int u = 0; u < U; ++u) cur[u] = nxt[u];
    }
  } else
  for (int64_t g = tid; g < a.G; g += NT) {
    Queue<KB> q[V];
#pragma unroll
    for (int e = 0; e < V; ++e) q[e].init();
    const uint8_t* colp = rowp + g * V * ESZ;
    const int64_t s_eff = (g < a.last_vec) ? s : s - 1;  // ragged final view-row
    for (int64_t t0 = 0; t0 < s_eff; t0 += U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t t = t0 + u;
        v[u] = (t < s_eff) ? ldg_stream(colp + t * b * ESZ) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t t = t0 + u;
        if (t < s_eff) {
          bad |= nonfinite_bits<DT>(v[u]);
          float f[V];
          unpack<DT>(v[u], f);
#pragma unroll
          for (int e = 0; e < V; ++e) q[e].push(f[e], (int)t);
        }
      }
    }
    spill_col(q, g);
  }
  if (tr) g_trace[blockIdx.x][2] = g_trace[blockIdx.x][3] = gtime();
  if (__syncthreads_or(nonfinite_hit<DT>(bad)) && tid == 0 && a.flag) atomicOr(a.flag, 1u);
  if constexpr (ITEMS == 32) {
    if (a.lsd_lowbit) {
      // large pool: stable in-place LSD (5-bit digits, per-thread counters)
      // over the bits above the bucket id — the pool is already in bucket-id
      // order — instead of the atomic-bucketing rank engine
      __shared__ uint32_t lws[NT / 32][16];
      __shared__ uint32_t ltot[32], ldex[32];
      __shared__ unsigned long long lvary;
      lsd::sort_desc_inplace<NT, 32, 5>(pool, (int)a.P, a.lsd_lowbit,
                                        reinterpret_cast<uint32_t*>(smem + a.aux_off), lws, ltot, ldex, &lvary);
      if (tr) g_trace[blockIdx.x][5] = gtime();
      pdl_wait_writes(a.early != 0);
      for (int64_t q = tid; q < a.k; q += NT)
        emit_comp<DT>(pool[lsd::pad32((int)q)], row * a.k + q, a.geo, a.out_vals, a.out_idx);
      if (tr) g_trace[blockIdx.x][4] = gtime();
      return;
    }
  }
  stage2_emit<DT, NT, ITEMS>(pool, smem + a.aux_off, a.P, a.k, a.lognb, row, a.geo, a.out_vals,
                            a.out_idx, a.trace != 0, a.early != 0);
  if (tr) g_trace[blockIdx.x][4] = gtime();
}

// ============================================================ stage-1 pool (vector columns)
// Stage 1 alone for the generic (pool in global memory) path when the pool
// is too large for one CTA (cfg5: b = 65536, k_b = 2 -> 131072 survivors
// per row).  Same per-thread vector-column scan as fused_wide, but one
// thread per column across the whole grid and all of a column's slots in
// flight at once; survivors go to pool[row][j*k_b + z] (btk_stage1.cu's
// layout), the input to K2.  HIST: also count the survivors per coarse
// bin (the top POOL_HBITS bits of the composite key) in shared memory and
// flush the CTA's counts to hist[row][bin] with global atomics — the
// chunked Stage 2 (btk_pool.cu) plans from it without re-reading the pool.
// A CTA covers `groups` consecutive 256-column groups of one row.
template <int DT, int KB, int U, bool HIST>
__global__ void __launch_bounds__(256) s1_vec(const void* __restrict__ x, int64_t row_stride,
                                              int64_t n, int64_t b, int64_t s, int64_t G,
                                              int last_vec, CompGeo geo,
                                              uint64_t* __restrict__ pool, uint32_t* flag,
                                              uint32_t* __restrict__ hist, int groups,
                                              const int* __restrict__ rowmask) {
  constexpr int V = Vec<DT>::V;
  constexpr int ESZ = VT<DT>::W / 8;
  constexpr int NBINS = HIST ? (1 << POOL_HBITS) : 1;
  __shared__ uint32_t sh[NBINS];
  const int64_t row = blockIdx.y;
  if (rowmask && rowmask[row] >= 0) return;  // row already handled (btk_xchg.cu fallback mask)
  const int hshift = geo.nbits - POOL_HBITS;
  uint32_t bad = 0;
  if constexpr (HIST) {
    for (int i = threadIdx.x; i < NBINS; i += 256) sh[i] = 0u;
    __syncthreads();
  }
  for (int grp = 0; grp < groups; ++grp) {
    const int64_t g = ((int64_t)blockIdx.x * groups + grp) * 256 + threadIdx.x;
    if (g < G) {
      const uint8_t* colp = static_cast<const uint8_t*>(x) + (row * row_stride + g * V) * ESZ;
      const int64_t s_eff = (g < last_vec) ? s : s - 1;
      Scanner<DT, KB> sc;
      sc.init();
      int64_t t0 = 0;
      for (; t0 + U <= s_eff; t0 += U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ldg_stream(colp + (t0 + u) * b * ESZ);
#pragma unroll
        for (int u = 0; u < U; ++u) sc.row(v[u], (int)(t0 + u));
      }
      for (; t0 < s_eff; ++t0) sc.row(ldg_stream(colp + t0 * b * ESZ), (int)t0);
      bad |= sc.nonfinite() ? 1u : 0u;
      uint64_t* dst = pool + row * b * KB;
      if constexpr (HIST) {
        sc.each_comp((int)g, b, 0, geo, [&](int64_t col, int z, uint64_t c) {
          dst[col * KB + z] = c;
          if (c) atomicAdd(&sh[(uint32_t)(c >> hshift)], 1u);
        });
      } else {
        sc.template spill<KB>(dst, (int)g, b, 0, geo);
      }
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0 && flag) atomicOr(flag, 1u);
  if constexpr (HIST) {
    uint32_t* hr = hist + row * NBINS;
    for (int i = threadIdx.x; i < NBINS; i += 256)
      if (sh[i]) atomicAdd(&hr[i], sh[i]);
  }
}

// ============================================================ planning
enum Kind { NONE = 0, NARROW = 1, WIDE = 2, ROWS = 3 };

struct Plan {
  Kind kind = NONE;
  int nt = 0;
  size_t smem = 0;
  size_t ws = 0;  // device workspace (none of the fused kernels needs one today)
  NarrowArgs na{};
  WideArgs wa{};
  RowsArgs ra{};
  int rows_gpl = 0, rows_items = 0;
};

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = NUM_SMS;
    n = v;
  }
  return n;
}

inline bool common_envelope(const Problem& p) {
  if (p.layout != 0 || p.kb > 8) return false;
  const int V = vec_of(p.dtype), esz = esz_of(p.dtype);
  if (V * p.kb > 32) return false;  // register queue budget (V buckets x k_b)
  if (p.b % V || p.n % V) return false;
  if ((reinterpret_cast<uintptr_t>(p.x) & 15) || ((p.row_stride * esz) & 15)) return false;
  if (p.b * p.kb > FUSED_POOL_CAP) return false;
  return true;
}

inline bool plan_narrow(const Problem& p, Plan& pl) {
  const int V = vec_of(p.dtype), esz = esz_of(p.dtype);
  const int64_t G = p.b / V, s = (p.n + p.b - 1) / p.b, P = p.b * p.kb;
  const int NT = env_int("BTK_NT", 0) == 256 ? 256 : (G <= 16 ? 128 : 256);
  if (G > NT) return false;
  NarrowArgs& a = pl.na;
  a.x = p.x; a.row_stride = p.row_stride;
  a.m = p.m; a.n = p.n; a.k = p.k; a.b = p.b; a.kb = p.kb; a.s = s;
  a.G = (int)G;
  a.R = (int)(NT / G);
  const int64_t vrow_bytes = p.b * esz;
  a.last_vec = (int)((p.n - (s - 1) * p.b) / V);
  a.P = P;
  a.sort_items = sort_items_for(P, NT);
  if (a.sort_items > 32) return false;  // engine keys per thread
  a.lognb = rank_lognb(P);
  // Launch shape (measured on B200, tools/sweep_narrow2.sh): rows of >= 1 MB
  // run one CTA per row with a deep ring (3 x 48 KB in flight; cfg3 94% of
  // the copy peak); shorter rows split over a cluster of S CTAs so about
  // two CTAs land per SM, each with >= 64 KB (cfg1: S = 2, 2 x 32 KB).
  const int64_t row_bytes = p.n * esz;
  const int nsm = num_sms();
  // With BTK_INPUT_READY (back-to-back independent batches) the next launch
  // streams into the SMs this one leaves idle, so when the rows alone cover
  // at least half the SMs one CTA per row wins: no cluster handoff, and
  // smaller stages (16 KB) get the first bytes in sooner (cfg1: 7.3 vs
  // 6.2 TB/s; without the flag the cluster split stays: 3.6 vs 2.4 TB/s).
  const bool early = (p.flags & 1u) && pdl_enabled();
  const bool solo = early && row_bytes < (1 << 20) && p.m >= nsm / 2;
  int S = 1;
  if (row_bytes < (1 << 20) && !solo) {
    while (S < 8 && p.m * (S * 2) <= 2 * (int64_t)nsm && row_bytes / (S * 2) >= 64 * 1024) S *= 2;
  }
  if (env_int("BTK_S", 0)) S = env_int("BTK_S", 0);
  while (S < 8 && (s + S - 1) / S >= 0xFFFF) S *= 2;  // 16-bit slot codes of the packed scanner
  if (S > s || (s + S - 1) / S >= 0xFFFF) return false;
  const int kbt = kb_tmpl(p.kb);
  const size_t scratch = (size_t)a.R * p.b * kbt * 8;
  const size_t regA = a16(scratch);
  // post-scan layout aliases the ring (scratch, pool, engine scratch); the
  // S partial slots the cluster CTAs push into live beyond both, because a
  // finished CTA may push while the leader is still streaming
  a.scratch_off = 0;
  a.pool_off = regA;
  a.aux_off = a.pool_off + (P <= 64 ? 64 * 8 : a16((size_t)P * 8));
  const size_t post = a.pool_off + stage2_bytes(P, p.k, NT);
  const size_t part_bytes = (size_t)S * p.b * kbt * 8;
  const bool deep = row_bytes / S >= (1 << 20);
  int NS = env_int("BTK_NS", deep ? 3 : 2);
  // (back-to-back launches also favour smaller stages on deep rows:
  // cfg3 3 x 32 KB 7.4 vs 3 x 48 KB 6.8 TB/s; serial launches keep 48 KB)
  int stage_kb = env_int("BTK_STAGE_KB", deep ? (early ? 32 : 48) : (solo ? 16 : 32));
  size_t smem = 0;
  for (;; stage_kb /= 2) {
    int64_t T = std::max<int64_t>(1, ((int64_t)stage_kb * 1024) / vrow_bytes);
    if (T >= a.R) T = (T / a.R) * a.R;
    if (T * vrow_bytes > 64 * 1024) return false;
    const int64_t stages = ((s + S - 1) / S + T - 1) / T;
    const int ns = (int)std::min<int64_t>(std::min<int64_t>(stages, NS), MAX_STAGES);
    const size_t part_off = a16(std::max(post, (size_t)ns * (size_t)(T * vrow_bytes)));
    const size_t sm = part_off + part_bytes;
    if (sm <= SMEM_LIMIT || stage_kb <= 8) {
      a.T = (int)T;
      a.stage_bytes = (size_t)(T * vrow_bytes);
      a.part_off = part_off;
      NS = ns;
      smem = sm;
      break;
    }
  }
  if (smem == 0 || smem > SMEM_LIMIT) return false;
  a.S = S;
  a.NS = NS;
  a.geo = p.geo;
  a.flag = p.flag;
  a.trace = env_int("BTK_TRACE", 0);
  a.early = early ? 1 : 0;
  pl.kind = NARROW;
  pl.nt = NT;
  pl.smem = smem;
  return true;
}

inline bool plan_wide(const Problem& p, Plan& pl) {
  const int V = vec_of(p.dtype), esz = esz_of(p.dtype);
  (void)esz;
  const int64_t G = p.b / V, s = (p.n + p.b - 1) / p.b, P = p.b * p.kb;
  WideArgs& a = pl.wa;
  a.x = p.x; a.row_stride = p.row_stride;
  a.m = p.m; a.n = p.n; a.k = p.k; a.b = p.b; a.kb = p.kb; a.s = s; a.G = G;
  a.P = P;
  a.last_vec = (int)((p.n - (s - 1) * p.b) / V);
  a.sort_items = sort_items_for(P, WIDE_NT);
  if (a.sort_items > 32) return false;
  a.lognb = rank_lognb(P);
  a.pool_off = 0;
  a.aux_off = P <= 64 ? 64 * 8 : a16((size_t)P * 8);
  a.geo = p.geo;
  a.flag = p.flag;
  a.trace = env_int("BTK_TRACE", 0);
  a.early = (p.flags & 1u) && pdl_enabled() ? 1 : 0;
  pl.smem = stage2_bytes(P, p.k, WIDE_NT);
  a.lsd_lowbit = 0;
  // opt-in (BTK_WIDE_LSD=1): measured slower than the rank engine at cfg2
  // (61.6 vs 43 us: fp32 owner keys vary in ~35 bits above the bucket id,
  // 7 five-bit passes)
  if (a.sort_items == 32 && env_int("BTK_WIDE_LSD", 0)) {
    // the pool is in bucket-id order: for b a power of two the low log2(b)
    // bits of the index field (~j) are already sorted
    int lb = 0;
    while ((int64_t(1) << lb) < p.b) ++lb;
    a.lsd_lowbit = ((p.b & (p.b - 1)) == 0) ? 1 + lb : 1;
    a.aux_off = a16((size_t)lsd::pad32((int)P) * 8);
    pl.smem = a.aux_off + (size_t)16 * WIDE_NT * 4;  // pool (padded) + 16 counter words per thread
  }
  pl.kind = WIDE;
  pl.nt = WIDE_NT;
  return pl.smem <= SMEM_LIMIT;
}

// One warp per row (fused_rows): many rows, b <= 64 vectors, pool <= 1024.
inline bool plan_rows(const Problem& p, Plan& pl) {
  const int V = vec_of(p.dtype);
  const int64_t G = p.b / V, s = (p.n + p.b - 1) / p.b, P = p.b * p.kb;
  if (p.kb != kb_tmpl(p.kb) || G > 64 || P > 1024 || s >= 0xFFFF) return false;
  if (V * p.kb > 16) return false;  // register queues per lane (see launch_rows)
  RowsArgs& a = pl.ra;
  a.x = p.x; a.row_stride = p.row_stride;
  a.m = p.m; a.n = p.n; a.k = p.k; a.b = p.b; a.kb = p.kb; a.s = s;
  a.G = (int)G;
  a.last_vec = (int)((p.n - (s - 1) * p.b) / V);
  a.P = P;
  a.lognb = std::min(rank_lognb(P), 8);
  a.inv_off = a16((size_t)std::max<int64_t>(P, 32) * 8);
  a.hist_off = a.inv_off + a16((size_t)p.k * 2);
  a.bid_off = a.hist_off + a16((size_t)((1 << a.lognb) + 2) * 4);
  a.warp_smem = a.bid_off + a16((size_t)std::max<int64_t>(P, 32) * 2);
  const size_t smem = 8 * a.warp_smem;
  if (smem > SMEM_LIMIT) return false;
  pl.rows_gpl = G <= 32 ? 1 : 2;
  pl.rows_items = P <= 256 ? 8 : (P <= 512 ? 16 : 32);
  a.geo = p.geo;
  a.flag = p.flag;
  a.early = (p.flags & 1u) && pdl_enabled() ? 1 : 0;
  pl.kind = ROWS;
  pl.nt = 256;
  pl.smem = smem;
  return true;
}

inline bool make_plan(const Problem& p, Plan& pl) {
  if (!common_envelope(p)) return false;
  const int want_rows = env_int("BTK_ROWS", -1);
  const bool rows = want_rows >= 0 ? want_rows != 0 : p.m >= 8 * (int64_t)num_sms();
  if (rows && plan_rows(p, pl)) return true;
  if (plan_narrow(p, pl)) return true;
  return plan_wide(p, pl);
}

template <int DT, int KB>
cudaError_t launch_narrow(const Plan& pl, cudaStream_t st) {
  const NarrowArgs& a = pl.na;
  void (*kern)(NarrowArgs);
  switch (a.sort_items) {
    case 0: kern = pl.nt == 128 ? fused_narrow<DT, KB, 128, 0> : fused_narrow<DT, KB, 256, 0>; break;
    case 2: kern = pl.nt == 128 ? fused_narrow<DT, KB, 128, 2> : fused_narrow<DT, KB, 256, 2>; break;
    case 8: kern = pl.nt == 128 ? fused_narrow<DT, KB, 128, 8> : fused_narrow<DT, KB, 256, 8>; break;
    default: kern = pl.nt == 128 ? fused_narrow<DT, KB, 128, 32> : fused_narrow<DT, KB, 256, 32>; break;
  }
  cudaError_t e = ensure_smem_attr((const void*)kern, pl.smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(a.m * a.S));
  cfg.blockDim = dim3(pl.nt);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[3];
  int na = 0;
  attr[na].id = cudaLaunchAttributeClusterDimension;
  attr[na].val.clusterDim.x = a.S;
  attr[na].val.clusterDim.y = 1;
  attr[na].val.clusterDim.z = 1;
  ++na;
  if (env_int("BTK_CLB", 1)) {  // load-balancing cluster placement: cfg1 +2.2% (BTK_CLB=0 disables)
    attr[na].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
    attr[na].val.clusterSchedulingPolicyPreference = cudaClusterSchedulingPolicyLoadBalancing;
    ++na;
  }
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int DT, int KB>
cudaError_t launch_wide(const Plan& pl, cudaStream_t st) {
  const WideArgs& a = pl.wa;
  void (*kern)(WideArgs);
  switch (a.sort_items) {
    case 0: kern = fused_wide<DT, KB, WIDE_NT, WIDE_U, 0>; break;
    case 2: kern = fused_wide<DT, KB, WIDE_NT, WIDE_U, 2>; break;
    case 8: kern = fused_wide<DT, KB, WIDE_NT, WIDE_U, 8>; break;
    default: kern = fused_wide<DT, KB, WIDE_NT, WIDE_U, 32>; break;
  }
  cudaError_t e = ensure_smem_attr((const void*)kern, pl.smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)a.m);
  cfg.blockDim = dim3(WIDE_NT);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int DT, int KB, int GPL, int ITEMS>
cudaError_t launch_rows_t(const Plan& pl, cudaStream_t st) {
  constexpr int U = (GPL == 1 ? 8 : 4) / (KB > 2 ? 2 : 1);
  auto kern = fused_rows<DT, KB, GPL, U, ITEMS>;
  cudaError_t e = ensure_smem_attr((const void*)kern, pl.smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, pl.nt, pl.smem);
  if (e != cudaSuccess) return e;
  const int64_t want = (pl.ra.m + 7) / 8;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)std::max(1, per_sm) * num_sms()));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(pl.nt);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, pl.ra);
}

template <int DT, int KB>
cudaError_t launch_rows(const Plan& pl, cudaStream_t st) {
  if constexpr (Vec<DT>::V * KB > 16) {
    return cudaErrorNotSupported;  // plan_rows never selects these (register budget)
  } else {
    if (pl.rows_gpl == 1) {
      if (pl.rows_items == 8) return launch_rows_t<DT, KB, 1, 8>(pl, st);
      if (pl.rows_items == 16) return launch_rows_t<DT, KB, 1, 16>(pl, st);
      return launch_rows_t<DT, KB, 1, 32>(pl, st);
    }
    if (pl.rows_items == 8) return launch_rows_t<DT, KB, 2, 8>(pl, st);
    if (pl.rows_items == 16) return launch_rows_t<DT, KB, 2, 16>(pl, st);
    return launch_rows_t<DT, KB, 2, 32>(pl, st);
  }
}

template <int DT, int KB>
cudaError_t launch_any(const Plan& pl, cudaStream_t st) {
  if (pl.kind == ROWS) return launch_rows<DT, KB>(pl, st);
  return pl.kind == NARROW ? launch_narrow<DT, KB>(pl, st) : launch_wide<DT, KB>(pl, st);
}

template <int DT>
cudaError_t launch_kb(const Plan& pl, int64_t kb, cudaStream_t st) {
  if (kb <= 1) return launch_any<DT, 1>(pl, st);
  if (kb <= 2) return launch_any<DT, 2>(pl, st);
  if (kb <= 4) return launch_any<DT, 4>(pl, st);
  if constexpr (DT == F32) return launch_any<DT, 8>(pl, st);
  return cudaErrorNotSupported;
}

}  // namespace fz
}  // namespace btk
