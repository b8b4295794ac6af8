// The exchange family for large pools (cfg5: 131072 survivors per row,
// k = 65536): Stage 1 + Stage 2 partitioned by value range over 16 owners
// per row, with no radix passes over the whole pool.  Two pipelines:
//
//   * the batched pipeline (xb_split / xb_part / xb_sort, below the cluster
//     kernel; the default for 16-bit dtypes): the same five steps as
//     ordinary launches over batches of rows, splitters from a sampling
//     pass, intermediates in global memory (~0.3 MB of keys per row);
//   * the cluster kernel (fused_xchg; BTK_XB=0, and fp32 with BTK_XC=1),
//     described here: one row per 16-CTA cluster in ONE launch, with no HBM
//     round trip for the candidates.  Its cluster barriers left ~70% of
//     each CTA's life waiting, hence the batched pipeline.
//
// Restates reference approx.py:208-282 (stage1 + topk_with_indices) and
// exact.py:130-159 (_canonical_order) for the B200: a cluster of C CTAs
// owns one row; the row's b buckets (interleaved: the columns of the row
// viewed as (s, b), approx.py:112-131) are split into C column ranges.
//
//   1. stage 1    CTA r streams its b/C columns (16-byte LDGs, all s
//                 view-rows of a vector column in flight) and keeps the top
//                 k_b (value, slot) per column in registers (strict ">" on
//                 ascending slots == first maximum, approx.py:151-162).  The
//                 survivors go to a shared-memory candidate array in column
//                 (= bucket id j) order.
//   2. splitters  every CTA ranks a strided sample of its candidates and
//                 stores its local quantiles (C-1 owner boundaries and a
//                 conservative selection threshold: the sample rank of k
//                 plus 4 sigma) into every CTA; after one barrier the CTAs
//                 average them, so each owner range holds ~k/C keys.  Only
//                 splitters come from the sample; every count below is
//                 exact.
//   3. exchange   each thread counts its (column-ordered) candidates per
//                 owner; block and cluster prefix sums give every candidate
//                 a stable slot in its owner's receive buffer, written with
//                 st.shared::cluster.  Arrival order is source rank, then
//                 column: every receive buffer is sorted by bucket id j.
//                 The exact per-owner totals give each owner its output
//                 offset; a row whose threshold kept < k keys or whose
//                 owner overflowed takes the fallback below.
//   4. sort       each owner sorts its keys descending with stable 4-bit
//                 LSD passes (per-thread packed counters, block scan), only
//                 over bits that vary, and never over the j bits: a key's
//                 index field is (~t | ~j) for idx = t*b + j (b a power of
//                 two) and the buffer already is in ascending-j order.
//   5. emit       the owner decodes its first min(count, k - start) keys
//                 into (value bits, int64 index) at its output offset.
//
// Fallback rows (partition overflow, or a 16-bit owner range too wide for
// 32-bit sort keys) go to a device-side list; xc_fallback recomputes them
// with per-CTA scratch (its CTAs exit at once when the list is empty).
//
// Keys: for 16-bit dtypes a candidate is a 32-bit record
// (vkey16 << 16 | (0x7FFF - t) << 1 | negzero) with j implied by its
// position, and the sort key is (comp - base_r) in 32 bits, base_r the
// owner's range floor aligned to the value field; fp32 uses the 64-bit
// composite key (btk_common.cuh) throughout.
#include <unordered_map>

#include "btk_fused_impl.cuh"
#include "btk_k2dev.cuh"

namespace btk {
namespace xc {
using namespace fz;

// --------------------------------------------------------------- DSMEM helpers
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ uint32_t ld_cl_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_cl_u64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_cl(uint32_t a, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cl(uint32_t a, uint64_t v) {
  asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  cluster_arrive_release();
  cluster_wait_acquire();
}

// padded record index: one record of padding per 128 bytes, so a thread's
// consecutive records (blocked layouts) are bank-conflict free
template <typename KT>
__host__ __device__ constexpr int padk(int p) {
  return sizeof(KT) == 4 ? p + (p >> 5) : p + (p >> 4);
}

constexpr int SPC = 128;  // sample keys per CTA

struct XArgs {
  const void* x;
  int64_t row_stride;
  int64_t m, n, k, b;
  int s, logb, cols, ncand;
  CompGeo geo;
  void* out_vals;
  int64_t* out_idx;
  uint32_t* flag;
  int* fb_count;   // rows whose partition overflowed (zeroed before the launch) ...
  int* fb_list;    // ... and their ids, finished by xc_fallback
  int trace;       // development timeline (BTK_XC_TRACE=1): globaltimer per CTA and phase
  int early;       // read the input before the predecessor completes (BTK_INPUT_READY)
};

constexpr int TRACE_CTAS = 16384;
static __device__ unsigned long long g_xtrace[TRACE_CTAS][8];
__device__ __forceinline__ void mark(const XArgs& a, int ph) {
  if (a.trace && threadIdx.x == 0 && blockIdx.x < TRACE_CTAS) g_xtrace[blockIdx.x][ph] = gtime();
}

// candidate record <-> composite key
template <typename KT>
__device__ __forceinline__ KT to_rec(uint64_t c, const XArgs& a) {
  if constexpr (sizeof(KT) == 8) {
    return c;
  } else {
    const uint32_t vk = (uint32_t)(c >> (a.geo.ib + 1));
    const uint32_t idx = a.geo.imax - (uint32_t)((c >> 1) & a.geo.imax);
    const uint32_t t = idx >> a.logb;
    return (vk << 16) | ((0x7FFFu - t) << 1) | (uint32_t)(c & 1u);
  }
}
template <typename KT>
__device__ __forceinline__ uint64_t from_rec(KT r, uint32_t j, const XArgs& a) {
  if constexpr (sizeof(KT) == 8) {
    return r;
  } else {
    const uint32_t t = 0x7FFFu - ((r >> 1) & 0x7FFFu);
    return make_comp(r >> 16, (t << a.logb) | j, r & 1u, a.geo);
  }
}

// Per-thread digit counters and the block digit scan: btk_lsd.cuh (4-bit
// digits here: 8 counter words per thread).
using lsd::count_digit;
using lsd::digit_base;
template <int NT>
__device__ __forceinline__ void digit_scan(uint32_t* cnt, uint32_t (*ws)[8], uint32_t* tot, uint32_t* dex) {
  lsd::digit_scan<NT, 8>(cnt, ws, tot, dex);
}

// Shared-memory carve-up (bytes), identical on host and device.
constexpr int LUTN = 8192;  // 16-bit owner table: vkeys above the threshold
template <typename KT, int NT, int IPT, int ITEMS>
struct Layout {
  static constexpr int CAP = NT * ITEMS;
  static constexpr size_t CAND = ((size_t)padk<KT>(NT * IPT) * sizeof(KT) + 127) / 128 * 128;
  static constexpr size_t BUF = ((size_t)padk<KT>(CAP) * sizeof(KT) + 127) / 128 * 128;
  static constexpr size_t A = 0;                 // candidates, later the sort's partner buffer
  static constexpr size_t B = A + (CAND > BUF ? CAND : BUF);  // receive buffer (the sample first)
  static constexpr size_t CNT = B + BUF;         // u32 [8][NT] digit counters / bases
  static constexpr size_t LUT = CNT + (size_t)NT * 8 * 4;  // u8 owner per vkey (16-bit dtypes)
  static constexpr size_t BYTES = LUT + (sizeof(KT) == 4 ? LUTN : 0);
};

template <int DT, int KB, int C, int NT, int IPT, int ITEMS, typename KT>
__global__ void __launch_bounds__(NT, 2) fused_xchg(XArgs a) {
  constexpr int V = Vec<DT>::V;
  constexpr int ESZ = VT<DT>::W / 8;
  constexpr int NW = NT / 32;
  constexpr int CAP = NT * ITEMS;
  constexpr int U = 8;  // 16-byte loads in flight per thread
  constexpr bool K32 = sizeof(KT) == 4;
  using L = Layout<KT, NT, IPT, ITEMS>;
  static_assert(C <= 16 && (C & (C - 1)) == 0, "cluster");
  static_assert(2 * SPC * 8 <= L::BUF, "sample fits the receive buffer");
  extern __shared__ __align__(128) uint8_t smem[];
  KT* cand = reinterpret_cast<KT*>(smem + L::A);
  KT* recv = reinterpret_cast<KT*>(smem + L::B);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + L::CNT);
  uint8_t* lut = smem + L::LUT;
  __shared__ uint32_t ws[NW][8];
  __shared__ uint32_t dtot[16], dex[16];
  __shared__ unsigned long long est[C][C + 1];   // every CTA's splitter estimates
  __shared__ unsigned long long lspl[C + 1];     // the splitters (identical in every CTA);
                                                 // 16-bit dtypes: vkeys, else comps
  __shared__ unsigned long long s_max, s_min;
  __shared__ uint32_t sendcnt[16], tot[C], dbase[C];
  __shared__ unsigned long long s_vary, s_start;
  __shared__ int s_why;

  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t rank = cta_rank();
  const int64_t row = blockIdx.x / C;
  const CompGeo geo = a.geo;
  const int64_t col0 = (int64_t)rank * a.cols;
  const int gv = a.cols / V;
  const int ib1 = geo.ib + 1;

  if (tid == 0) { s_max = 0ull; s_min = ~0ull; s_vary = 0ull; }
  if (tid < C) { tot[tid] = 0u; dbase[tid] = 0u; }
  __syncthreads();
  // every CTA of the cluster must have started before any DSMEM access: arrive
  // now, wait right before the first remote store (stage 1 hides the latency)
  cluster_arrive_release();
  pdl_trigger();
  if (!a.early) pdl_wait();
  mark(a, 0);

  // ---------------------------------------------------------------- 1. stage 1
  {
    uint32_t bad = 0;
    uint64_t mx = 0ull, mn = ~0ull;
    const uint8_t* rowp = static_cast<const uint8_t*>(a.x) + (row * a.row_stride + col0) * ESZ;
    const int64_t vstride = a.b * ESZ;
    for (int g = tid; g < gv; g += NT) {
      Scanner<DT, KB> sc;
      sc.init();
      const uint8_t* colp = rowp + (int64_t)g * V * ESZ;
      for (int t0 = 0; t0 < a.s; t0 += U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          v[u] = (t0 + u < a.s) ? ldg_stream(colp + (int64_t)(t0 + u) * vstride) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (t0 + u < a.s) sc.row(v[u], t0 + u);
      }
      bad |= sc.nonfinite() ? 1u : 0u;
      sc.each_comp((int)(col0 / V) + g, a.b, 0, geo, [&](int64_t col, int z, uint64_t c) {
        cand[padk<KT>((int)((col - col0) * KB + z))] = to_rec<KT>(c, a);
        mx = c > mx ? c : mx;
        mn = c < mn ? c : mn;
      });
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const uint64_t x1 = __shfl_xor_sync(0xFFFFFFFFu, mx, o), x2 = __shfl_xor_sync(0xFFFFFFFFu, mn, o);
      mx = x1 > mx ? x1 : mx;
      mn = x2 < mn ? x2 : mn;
    }
    if (lane == 0) {
      atomicMax(&s_max, (unsigned long long)mx);
      atomicMin(&s_min, (unsigned long long)mn);
    }
    if (__syncthreads_or(bad) && tid == 0 && a.flag) atomicOr(a.flag, 1u);
  }
  mark(a, 1);

  // ---------------------------------------------------------------- 2. splitters
  // Every CTA ranks a strided sample of SPC of its candidates (count of
  // larger samples; comps are unique), takes its local quantiles at the
  // owner boundaries and at the threshold rank, and stores them into every
  // CTA; after one barrier each CTA averages the C estimates per splitter
  // (identical data -> identical splitters in every CTA).  The averages
  // are ordered because every CTA's quantiles are.  For 16-bit dtypes the
  // splitters are then rounded down to whole values (vkeys), so a key's
  // owner is a table lookup on its vkey.
  int rthr = SPC;  // local sample rank of the threshold (k plus 4 sigma of the pooled sample)
  {
    const double q = (double)a.k / ((double)a.b * KB);
    if (q < 1.0) {
      const double r = SPC * q + 4.0 * sqrt(SPC * q * (1.0 - q) / C) + 0.5;
      rthr = r >= (double)SPC ? SPC : (int)ceil(r);
    }
  }
  const bool select_all = rthr >= SPC;
  {
    uint64_t* smp = reinterpret_cast<uint64_t*>(smem + L::B);  // SPC sampled comps
    uint64_t* srt = smp + SPC;                                   // ranked
    if (tid < SPC) {
      const int stride = a.ncand / SPC;
      // the in-stride offset varies with tid (odd step) so the sample covers
      // every queue slot z = p % k_b, not one aliased slot
      const int p = tid * stride + (int)(((uint64_t)row * 40503u + rank * 977u + tid * 7u) % (uint64_t)stride);
      smp[tid] = from_rec<KT>(cand[padk<KT>(p)], (uint32_t)(col0 + p / KB), a);
    }
    __syncthreads();
    if (tid < SPC) {
      const uint64_t x = smp[tid];
      int r = 0;
#pragma unroll 8
      for (int q = 0; q < SPC; ++q) r += smp[q] > x ? 1 : 0;
      srt[r] = x;
    }
    __syncthreads();
    cluster_wait_acquire();  // all peers resident (matches the arrive above)
    if (tid <= C) {  // local estimate of splitter tid, stored into every CTA
      uint64_t v;
      if (tid == 0) v = s_max;
      else if (tid < C) v = srt[(tid * rthr) / C];
      else v = select_all ? s_min : srt[rthr];
      const uint32_t dst = smem_u32(&est[rank][tid]);
#pragma unroll 4
      for (int r = 0; r < C; ++r) st_cl(mapa(dst, (uint32_t)r), v);
    }
  }
  cluster_sync_all();  // A: every CTA's estimates everywhere
  mark(a, 2);
  if (tid <= C) {
    uint64_t v;
    if (tid == 0) {  // the cluster's max + 1 (exact)
      v = est[0][0];
      for (int r = 1; r < C; ++r) v = est[r][0] > v ? est[r][0] : v;
      v = K32 ? (v >> ib1) + 1ull : v + 1ull;
    } else if (tid == C && select_all) {  // the cluster's min (exact): everything is selected
      v = est[0][C];
      for (int r = 1; r < C; ++r) v = est[r][C] < v ? est[r][C] : v;
      if (K32) v >>= ib1;
    } else {
      uint64_t sum = 0;
      for (int r = 0; r < C; ++r) sum += est[r][tid];
      v = sum / C;
      if (K32) v >>= ib1;
    }
    lspl[tid] = v;
  }
  __syncthreads();
  // 16-bit dtypes: owner table over the selected vkeys [lspl[C], lspl[0])
  const uint32_t vthr = (uint32_t)lspl[C];
  const uint32_t vspan = K32 ? (uint32_t)(lspl[0] - lspl[C]) : 0u;
  const uint32_t vlim = vspan <= (uint32_t)LUTN ? vspan : 0u;  // too wide: fallback row
  if constexpr (K32) {
    if (vspan <= (uint32_t)LUTN) {
      for (uint32_t i = tid; i < vspan; i += NT) {
        const uint64_t v = vthr + i;
        uint32_t o = 0;
#pragma unroll
        for (int c = 1; c < C; ++c) o += lspl[c] > v ? 1u : 0u;
        lut[i] = (uint8_t)o;
      }
    }
    __syncthreads();
  }
  mark(a, 3);

  // ---------------------------------------------------------------- 3. exchange
  // owner of a candidate: #{c in 1..C : spl[c] > key}; C = below the threshold
  auto owner = [&](KT rec, uint32_t j) -> uint32_t {
    if constexpr (K32) {
      const uint32_t off = (rec >> 16) - vthr;  // wraps for vkeys below the threshold
      return off < vlim ? (uint32_t)lut[off] : (uint32_t)C;
    } else {
      const uint64_t x = rec;
      uint32_t o = 0;  // largest o with spl[o] > x (spl[0] exceeds every key)
#pragma unroll
      for (int st = C / 2; st > 0; st >>= 1)
        if (x < lspl[o + st]) o += st;
      if (x < lspl[C]) o = C;
      return o;
    }
  };
  // 32-bit sort key of a candidate for owner d: value offset above the
  // owner's lowest vkey, then the complemented index, then negzero
  auto key32 = [&](KT rec, uint32_t j, uint32_t d) -> uint32_t {
    const uint32_t t = 0x7FFFu - ((rec >> 1) & 0x7FFFu);
    const uint32_t idx = (t << a.logb) | j;
    return (((uint32_t)(rec >> 16) - (uint32_t)lspl[d + 1]) << ib1) | ((geo.imax - idx) << 1) | (uint32_t)(rec & 1u);
  };
  const int p0 = tid * IPT;
  uint32_t dl[IPT];
#pragma unroll
  for (int q = 0; q < 8; ++q) cnt[q * NT + tid] = 0u;
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int p = p0 + i;
    uint32_t d = (uint32_t)C;
    if (p < a.ncand) d = owner(cand[padk<KT>(p)], (uint32_t)(col0 + p / KB));
    dl[i] = d << 16;
    if (d < (uint32_t)C) dl[i] |= count_digit<NT>(cnt, d);
  }
  digit_scan<NT>(cnt, ws, sendcnt, dex);
  cluster_sync_all();  // C: send counts of every CTA published
  mark(a, 4);
  if (tid < C * C) {  // totals per owner and this CTA's base in each owner
    const int r = tid / C, d = tid % C;
    const uint32_t v = ld_cl_u32(mapa(smem_u32(&sendcnt[d]), (uint32_t)r));
    if (v) {
      atomicAdd(&tot[d], v);
      if ((uint32_t)r < rank) atomicAdd(&dbase[d], v);
    }
  }
  __syncthreads();
  if (tid == 0) {  // fallback verdict, output offset and receive count (one thread)
    uint64_t sum = 0, st = 0;
    int why = 0;  // fallback reasons: 1 owner overflow, 2 key range, 4 threshold kept < k
    for (int d = 0; d < C; ++d) {
      if ((uint32_t)d < rank) st += tot[d];
      sum += tot[d];
      if (tot[d] > (uint32_t)CAP) why |= 1;
      // the owner's value offsets must fit the 32-bit key above the index field
      if (K32 && tot[d] && ((lspl[d] - 1ull - lspl[d + 1]) >> (32 - ib1)) != 0ull) why |= 2;
    }
    if (K32 && vspan > (uint32_t)LUTN) why |= 2;
    if (sum < (uint64_t)a.k) why |= 4;
    s_start = st;
    s_why = why;
  }
  __syncthreads();
  const int64_t start = (int64_t)s_start;
  const int R = (int)tot[rank];
  pdl_wait_writes(a.early != 0);  // first global writes below
  if (s_why) {  // identical verdict in every CTA (same splitters, same totals)
    if (rank == 0 && tid == 0) a.fb_list[atomicAdd(a.fb_count, 1)] = (int)row;
    cluster_sync_all();  // peers may still read this CTA's send counts
    return;
  }
  {
    const uint32_t recv_s = smem_u32(recv);
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const uint32_t d = dl[i] >> 16;
      if (d < (uint32_t)C) {
        const int p = p0 + i;
        const KT rec = cand[padk<KT>(p)];
        const uint32_t j = (uint32_t)(col0 + p / KB);
        const uint32_t pos = dbase[d] + digit_base<NT>(cnt, d) + (dl[i] & 0xFFFFu);
        const uint32_t dst = mapa(recv_s + (uint32_t)padk<KT>((int)pos) * (uint32_t)sizeof(KT), d);
        if constexpr (K32) st_cl(dst, key32(rec, j, d));
        else st_cl(dst, (uint64_t)rec);
      }
    }
  }
  cluster_sync_all();  // D: every receive buffer complete; no remote traffic after this
  mark(a, 5);

  // ---------------------------------------------------------------- 4. sort
  const int items = (R + NT - 1) / NT;
  {
    KT vary = 0;
    const KT k0 = R ? recv[0] : (KT)0;
    for (int p = tid; p < items * NT; p += NT) {
      if (p < R) vary |= recv[padk<KT>(p)] ^ k0;
      else recv[padk<KT>(p)] = (KT)0;  // pads sort last
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) vary |= __shfl_xor_sync(0xFFFFFFFFu, vary, o);
    if (lane == 0 && vary) atomicOr(&s_vary, (unsigned long long)vary);
  }
  __syncthreads();
  KT* src = recv;
  KT* dst = cand;
  {
    constexpr int KBITS = (int)sizeof(KT) * 8;
    const KT vary = (KT)s_vary;
    const int lowbit = 1 + a.logb;  // negzero and j bits: already in order
    for (int shift = lowbit; shift < KBITS && (vary >> shift) != 0; shift += 4) {
      if (((vary >> shift) & (KT)0xF) == 0) continue;
      uint32_t sl[ITEMS];
#pragma unroll
      for (int q = 0; q < 8; ++q) cnt[q * NT + tid] = 0u;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        if (i < items) {
          const KT key = src[padk<KT>(tid * items + i)];
          const uint32_t d = 15u - (uint32_t)((key >> shift) & (KT)0xF);
          sl[i] = (d << 16) | count_digit<NT>(cnt, d);
        }
      }
      digit_scan<NT>(cnt, ws, dtot, dex);
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        if (i < items) {
          const uint32_t d = sl[i] >> 16;
          const int r = (int)(dex[d] + digit_base<NT>(cnt, d) + (sl[i] & 0xFFFFu));
          dst[padk<KT>(r)] = src[padk<KT>(tid * items + i)];
        }
      }
      __syncthreads();
      KT* t = src; src = dst; dst = t;
    }
  }

  // ---------------------------------------------------------------- 5. emit
  mark(a, 6);
  const int keep = (int)min((int64_t)R, a.k - start);
  for (int q = tid; q < keep; q += NT) {
    const KT key = src[padk<KT>(q)];
    uint64_t c;
    if constexpr (K32) {
      c = ((uint64_t)((uint32_t)lspl[rank + 1] + (key >> ib1)) << ib1) | (uint64_t)(key & ((1u << ib1) - 1u));
    } else {
      c = key;
    }
    emit_comp<DT>(c, row * a.k + start + q, geo, a.out_vals, a.out_idx);
  }
  mark(a, 7);
}

// ================================================================ fallback
// Rows whose value partition overflowed (massive ties, or 16-bit owner
// ranges too wide for 32-bit keys), one CTA per row from a persistent grid
// over the device-side list: Stage 1 of the row again (same scanners) into
// the CTA's scratch slot, the MSD radix select of the k largest, a stable
// LSD through the slot, emit.  Scratch is per CTA, not per row: the
// workspace no longer grows with m (cfg5: 0.23 GB instead of 12.9 GB).
constexpr int FB_CTAS = 148;
constexpr int FB_NT = 512;

template <int DT, int KB>
__global__ void __launch_bounds__(FB_NT) xc_fallback(XArgs a, uint64_t* __restrict__ slots, int64_t slot_stride) {
  constexpr int V = Vec<DT>::V;
  constexpr int ESZ = VT<DT>::W / 8;
  constexpr int U = 8;
  const int cnt = *a.fb_count;
  if ((int)blockIdx.x >= cnt) return;
  const int tid = threadIdx.x;
  const int64_t P = a.b * KB;
  uint64_t* pool = slots + (int64_t)blockIdx.x * slot_stride;  // P keys
  uint64_t* sel = pool + P;                                     // k keys
  const int gv = (int)(a.b / V);
  for (int i = blockIdx.x; i < cnt; i += gridDim.x) {
    const int64_t row = a.fb_list[i];
    const uint8_t* rowp = static_cast<const uint8_t*>(a.x) + row * a.row_stride * ESZ;
    const int64_t vstride = a.b * ESZ;
    for (int g = tid; g < gv; g += FB_NT) {
      Scanner<DT, KB> sc;
      sc.init();
      const uint8_t* colp = rowp + (int64_t)g * V * ESZ;
      for (int t0 = 0; t0 < a.s; t0 += U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          v[u] = (t0 + u < a.s) ? ldg_stream(colp + (int64_t)(t0 + u) * vstride) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (t0 + u < a.s) sc.row(v[u], t0 + u);
      }
      sc.each_comp(g, a.b, 0, a.geo, [&](int64_t col, int z, uint64_t c) { pool[col * KB + z] = c; });
    }
    __syncthreads();
    uint32_t bad = 0;  // non-finite input was flagged by the cluster kernel
    select_compact<FB_NT>(CompSource{pool}, P, a.k, sel, a.geo.nbits, bad);
    __syncthreads();
    const uint64_t* res = global_lsd<FB_NT, 8>(sel, pool, a.k, a.geo.nbits);
    for (int64_t q = tid; q < a.k; q += FB_NT) emit<DT>(res[q], row * a.k + q, a.geo, a.out_vals, a.out_idx);
    __syncthreads();
  }
}

template <int DT>
cudaError_t launch_fallback(const XArgs& a, int64_t kb, uint64_t* slots, int64_t slot_stride, cudaStream_t st) {
  const unsigned grid = (unsigned)std::min<int64_t>(a.m, FB_CTAS);
  switch (kb) {
    case 1: xc_fallback<DT, 1><<<grid, FB_NT, 0, st>>>(a, slots, slot_stride); break;
    case 2: xc_fallback<DT, 2><<<grid, FB_NT, 0, st>>>(a, slots, slot_stride); break;
    case 4: xc_fallback<DT, 4><<<grid, FB_NT, 0, st>>>(a, slots, slot_stride); break;
    default:
      if constexpr (DT == F32) {
        xc_fallback<DT, 8><<<grid, FB_NT, 0, st>>>(a, slots, slot_stride);
        break;
      }
      return cudaErrorNotSupported;
  }
  return cudaGetLastError();
}

// ================================================================ batched pipeline
// The same algorithm without clusters, for 16-bit dtypes (the default for
// them; BTK_XB=0 selects the cluster kernel above).  The splitters come from
// a sampling pass, so the chunks of a row never synchronise with each other:
// no cluster barriers, and the owner sorts run as independent, fully
// occupied CTAs.  Rows go in batches of up to 148; a batch's partition and
// sort are two launches, the sorts on a side stream over double-buffered
// sub-slots so batch i's sort can overlap batch i+1's partition.
//
//   xb_split   one CTA per row (all rows, once): Stage 1 of sample sites of
//              64 contiguous bytes per view-row (~1.6% of the row) gives SPC
//              sampled candidates per chunk of b/C columns; local quantiles
//              at the owner boundaries (fractional ranks, interpolated) and
//              at the threshold rank, averaged over the C chunks and rounded
//              down to fine keys (vkey << TB | top TB bits of the complemented
//              view-row; TB as large as keeps the owner table <= LUTN).
//   xb_part    grid (C, BR) per batch: CTA (c, r) runs Stage 1 on chunk c of
//              row r with the candidates in registers, assigns each its
//              owner (fine keys >= spl[1]: owner 0; else a table lookup;
//              below the threshold: none) and scatters the 32-bit sort keys
//              into its own sub-slot of each owner, stably (bucket order),
//              with the per-owner counts and the chunk's max vkey.
//   xb_sort    grid (C, BR) per batch: owner d of row r reads the C x (C+1)
//              counts, derives the row's verdict and its output offset (the
//              same in every CTA of the row), gathers its C sub-slots in
//              chunk order into registers, sorts them (4-bit LSD over the
//              bits above the bucket id) and emits.  Rows whose verdict fails
//              (sub-slot or owner overflow, key range, fewer than k kept) go
//              to the fallback list, finished by xc_fallback after the last
//              batch.
constexpr int XB_C = 16;       // chunks (= owners) per row
constexpr int XB_NT = 512;     // threads of every xb CTA
constexpr int XB_CAP = 8192;   // keys per owner in xb_sort (SNT x ITEMS)
constexpr int XB_SNT = 512;    // threads of an owner sort (256 x 32 items: fewer scan
                               // instructions but 80 registers, lower occupancy: slower)
constexpr int XB_ITEMS = XB_CAP / XB_SNT;
constexpr int XB_SMIN = 2;     // resident sorts per SM (64 registers)

__host__ __device__ inline int xb_rthr(int64_t k, int64_t P) {
  const double q = (double)k / (double)P;
  if (q >= 1.0) return SPC;
  const double r = SPC * q + 4.0 * sqrt(SPC * q * (1.0 - q) / XB_C) + 0.5;
  return r >= (double)SPC ? SPC : (int)ceil(r);
}

struct XBArgs {
  XArgs x;             // problem, outputs, fallback list
  int64_t r0;          // first row of the batch
  int br;              // rows in the batch
  int capc;            // keys per (owner, chunk) sub-slot
  uint32_t* spl;       // m x (C+1) splitter vkeys (spl[r][0] unused)
  uint32_t* seg;       // br x C owners x C chunks x capc sort keys
  uint32_t* cnt;       // br x C chunks x (C+1): per-owner counts, chunk max vkey
  size_t seg_elems, cnt_elems;  // one buffer of each (two with the side stream)
};

template <int DT, int KB>
__global__ void __launch_bounds__(XB_NT) xb_split(XBArgs A) {
  constexpr int V = Vec<DT>::V;
  constexpr int ESZ = VT<DT>::W / 8;
  constexpr int C = XB_C, NT = XB_NT;
  constexpr int G = SPC / (V * KB);  // sampled column groups per chunk
  static_assert(G >= 1 && G * V * KB == SPC, "sample layout");
  const XArgs& a = A.x;
  const int tid = threadIdx.x;
  const int64_t row = blockIdx.x;
  const int ib1 = a.geo.ib + 1;
  __shared__ unsigned long long smp[C][SPC];
  __shared__ unsigned long long srt[C][SPC];
  __shared__ unsigned long long est[C][C + 1];
  pdl_trigger();
  if (!a.early) pdl_wait();
  // sample sites of GS adjacent vector groups (64 contiguous bytes per
  // view-row: whole DRAM bursts, not one 16-byte piece per burst), NS sites
  // spread over the chunk at pseudo-random offsets
  constexpr int GS = G < 4 ? G : 4, NS = G / GS;
  const int span = a.cols / NS;  // columns between sites (multiple of GS * V)
  if (tid < C * G) {
    const int c = tid / G, g = tid % G, site = g / GS, w = g % GS;
    const int off = (int)(((uint64_t)row * 40503u + c * 977u + site * 7u) % (uint64_t)(span / (GS * V))) * (GS * V);
    const int64_t col = (int64_t)c * a.cols + (int64_t)site * span + off + w * V;
    const uint8_t* colp = static_cast<const uint8_t*>(a.x) + (row * a.row_stride + col) * ESZ;
    Scanner<DT, KB> sc;
    sc.init();
    // 8 loads in flight per thread (one latency per 8 view-rows, not per row)
    const uint32_t vs = (uint32_t)(a.b * ESZ);
    int t0 = 0;
    for (; t0 + 8 <= a.s; t0 += 8) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = ldg_stream(colp + (uint32_t)(t0 + u) * vs);
#pragma unroll
      for (int u = 0; u < 8; ++u) sc.row(v[u], t0 + u);
    }
    for (; t0 < a.s; ++t0) sc.row(ldg_stream(colp + (uint32_t)t0 * vs), t0);
    sc.each_comp((int)(col / V), a.b, 0, a.geo, [&](int64_t cc, int z, uint64_t comp) {
      smp[c][g * V * KB + (int)(cc - col) * KB + z] = comp;
    });
  }
  __syncthreads();
  for (int i = tid; i < C * SPC; i += NT) {
    const int c = i / SPC;
    const unsigned long long x = smp[c][i % SPC];
    int r = 0;
#pragma unroll 8
    for (int q = 0; q < SPC; ++q) r += smp[c][q] > x ? 1 : 0;
    srt[c][r] = x;
  }
  __syncthreads();
  const int rthr = xb_rthr(a.k, a.b * KB);
  for (int i = tid; i < C * C; i += NT) {
    const int c = i / C, q = 1 + i % C;
    if (q < C) {  // local quantile at the fractional rank q * rthr / C (linear in comp space)
      const int p256 = (q * rthr * 256) / C;
      const int r0 = p256 >> 8, f = p256 & 255;
      const unsigned long long hi = srt[c][r0], lo = srt[c][r0 + 1 < SPC ? r0 + 1 : r0];
      est[c][q] = hi - (((hi - lo) * (unsigned long long)f) >> 8);
    } else {
      est[c][q] = srt[c][rthr < SPC ? rthr : SPC - 1];
    }
  }
  __syncthreads();
  // Splitters are "fine keys": the value key with the top TB bits of the
  // view-row below it, fk = vkey << TB | (2^TB - 1 - (t >> (tbits - TB))),
  // ordered like the composite keys.  Whole values alone are too coarse
  // when one 16-bit value holds a large share of an owner's keys; TB is the
  // most view-row bits for which the owner table over [spl[C], spl[1])
  // still fits LUTN entries.
  __shared__ unsigned long long avg[C + 1];
  __shared__ int s_tb;
  if (tid > 0 && tid <= C) {
    unsigned long long sum = 0;
    for (int c = 0; c < C; ++c) sum += est[c][tid];
    avg[tid] = sum / C;
  }
  __syncthreads();
  const int tbits = a.geo.ib - a.logb;  // view-row bits of any index field
  if (tid == 0) {
    const uint32_t vspan = (uint32_t)(avg[1] >> ib1) - (uint32_t)(avg[C] >> ib1) + 1u;
    int tb = tbits;
    while (tb > 0 && ((uint64_t)vspan << tb) > (uint64_t)LUTN) --tb;
    s_tb = tb;
  }
  __syncthreads();
  pdl_wait_writes(a.early != 0);
  if (tid <= C) {
    const int tb = s_tb;
    uint32_t v = (uint32_t)tb;  // slot 0: TB
    if (tid > 0) {
      const unsigned long long c = avg[tid];
      const uint32_t idx = a.geo.imax - (uint32_t)((c >> 1) & a.geo.imax);
      v = ((uint32_t)(c >> ib1) << tb) | (((1u << tb) - 1u) - ((idx >> a.logb) >> (tbits - tb)));
    }
    A.spl[row * (C + 1) + tid] = v;
  }
}

// survivors of one scanned column group as (item, vkey, view-row, negzero);
// item = column offset in the group * KB + z
template <int DT, int KB, class F>
__device__ __forceinline__ void xb_each_rec(const Scanner<DT, KB>& sc, int g, const XArgs& a, F&& f) {
  if constexpr (DT != F32 && KB <= 2) {
    sc.each_raw([&](int i, uint32_t raw, uint32_t code) {
      f(i, vkey<DT>(raw), code, is_negzero<DT>(raw), code != 0xFFFFu);
    });
  } else {
    constexpr int V = Vec<DT>::V;
    sc.each_comp(g, a.b, 0, a.geo, [&](int64_t col, int z, uint64_t c) {
      const uint32_t idx = a.geo.imax - (uint32_t)((c >> 1) & a.geo.imax);
      f((int)(col - (int64_t)g * V) * KB + z, (uint32_t)(c >> (a.geo.ib + 1)), idx >> a.logb, (uint32_t)(c & 1u),
        c != 0ull);
    });
  }
}

// ST (s <= 16 view-rows): the view-row takes 4 record bits, so the owner
// fits in the record too and is not looked up a second time
template <int DT, int KB, bool ST>
__global__ void __launch_bounds__(XB_NT, 2) xb_part(XBArgs A) {
  constexpr int V = Vec<DT>::V;
  constexpr int ESZ = VT<DT>::W / 8;
  constexpr int C = XB_C, NT = XB_NT, NW = NT / 32;
  constexpr int IT = V * KB;  // survivors per column group (one group per thread and round)
  constexpr int U = KB >= 2 ? 4 : 8;  // 16-byte loads in flight (register budget of 64)
  const XArgs& a = A.x;
  const int tid = threadIdx.x, lane = tid & 31;
  const int c = blockIdx.x, rl = blockIdx.y;
  const int64_t row = A.r0 + rl;
  const int64_t col0 = (int64_t)c * a.cols;
  const int gv = a.cols / V;
  const int ib1 = a.geo.ib + 1;
  extern __shared__ __align__(128) uint8_t xsm[];
  uint32_t* cnt = reinterpret_cast<uint32_t*>(xsm);  // [8][NT] digit counters
  __shared__ uint8_t lut[LUTN];
  __shared__ uint32_t ws[NW][8];
  __shared__ uint32_t sendcnt[16], dex[16], run[16];
  __shared__ uint32_t lspl[C + 1], kofs[C];
  __shared__ uint32_t s_max;
  if (tid == 0) s_max = 0u;
  if (tid < 16) run[tid] = 0u;
  pdl_trigger();
  if (!a.early) pdl_wait();
  uint32_t bad = 0, mx = 0;
  uint32_t vthr = 0, tmax = 0;
  int tb = 0, tsh = 0;
  const uint8_t* rowp = static_cast<const uint8_t*>(a.x) + (row * a.row_stride + col0) * ESZ;
  const int64_t vstride = a.b * ESZ;
  uint32_t* seg = A.seg + ((int64_t)rl * C * C + c) * A.capc;  // + owner * C * capc
  const uint32_t ostride = (uint32_t)(C * A.capc);  // owner stride in the row-chunk's sub-slots
  const uint32_t capc = (uint32_t)A.capc;
  const int lb1 = a.logb + 1;
  for (int g0 = 0; g0 < gv; g0 += NT) {  // rounds: groups g0 + tid, in bucket order
    const int g = g0 + tid;
    const bool act = g < gv;
    // ---- Stage 1 of one column group (V buckets) in registers
    Scanner<DT, KB> sc;
    sc.init();
    if (act) {
      // 32-bit row offsets (s * b * ESZ < 4 GB): one pointer, no 64-bit
      // address arithmetic per load
      const uint8_t* colp = rowp + (int64_t)g * V * ESZ;
      const uint32_t vs = (uint32_t)vstride;
      int t0 = 0;
      for (; t0 + U <= a.s; t0 += U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ldg_stream(colp + (uint32_t)(t0 + u) * vs);
#pragma unroll
        for (int u = 0; u < U; ++u) sc.row(v[u], t0 + u);
      }
      for (; t0 < a.s; ++t0) sc.row(ldg_stream(colp + (uint32_t)t0 * vs), t0);
      bad |= sc.nonfinite() ? 1u : 0u;
    }
    // every bucket has >= k_b survivors (planner: s >= k_b), so an active
    // thread's items are all real
    uint32_t rec[IT];  // vkey << 16 | (rank among the thread's items of its owner) << 11 | view-row << 1 | negzero
    xb_each_rec<DT, KB>(sc, (int)(col0 / V) + g, a, [&](int i, uint32_t vk, uint32_t t, uint32_t nz, bool) {
      rec[i] = (vk << 16) | (t << 1) | nz;
      mx = act && vk > mx ? vk : mx;
    });
    if (g0 == 0) {
      // the splitters (xb_split) and this batch's buffers (the previous
      // batch's sort) are ready once the predecessor completed
      pdl_wait_writes(a.early != 0);
      if (tid <= C) lspl[tid] = A.spl[row * (C + 1) + tid];
      __syncthreads();
      tb = (int)lspl[0];
      tsh = a.geo.ib - a.logb - tb;
      tmax = (1u << tb) - 1u;
      // owner table over fine keys [spl[C], spl[C] + LUTN): owners 1..C-1
      // below spl[1], owner 0 from spl[1] up (beyond the table: owner 0 too)
      vthr = lspl[C];
      const uint32_t vspan = lspl[1] - lspl[C];
      for (uint32_t w = tid; w < (uint32_t)LUTN / 4; w += NT) {
        uint32_t word = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t i = 4 * w + e;
          uint32_t o = 0;
          if (i < vspan) {
            const uint32_t v = vthr + i;
            o = 1;
#pragma unroll
            for (int q = 2; q < C; ++q) o += lspl[q] > v ? 1u : 0u;
          }
          word |= o << (8 * e);
        }
        reinterpret_cast<uint32_t*>(lut)[w] = word;
      }
      if (tid < C) kofs[tid] = (lspl[tid + 1] >> tb) << ib1;
    }
    // ---- owners, stable ranks (thread-blocked items), scatter into sub-slots.
    // The item's rank among the thread's earlier items of its owner goes to
    // bits 11..15 of its record (view-rows < 1024); the owner is looked up
    // again after the scan (no second per-item register array).
    auto owner = [&](uint32_t r, bool ok) -> uint32_t {
      const uint32_t vk = ((r >> 16) << tb) | (tmax - (((r >> 1) & (ST ? 15u : 0x3FFu)) >> tsh));  // fine key
      const uint32_t off = vk - vthr;  // wraps below the threshold
      uint32_t d = vk < vthr ? (uint32_t)C : 0u;
      if (off < (uint32_t)LUTN) d = lut[off];
      return ok ? d : (uint32_t)C;
    };
#pragma unroll
    for (int q = 0; q < 8; ++q) cnt[q * NT + tid] = 0u;
    __syncthreads();  // table built; counters of the previous round consumed
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const uint32_t d = owner(rec[i], act);
      if constexpr (ST) {  // vkey << 16 | owner << 10 | rank << 5 | view-row << 1 | negzero
        rec[i] |= d << 10;
        if (d < (uint32_t)C) rec[i] |= lsd::count_digit<NT>(cnt, d) << 5;
      } else {
        if (d < (uint32_t)C) rec[i] |= lsd::count_digit<NT>(cnt, d) << 11;
      }
    }
    lsd::digit_scan_from<NT, 8>(cnt, ws, sendcnt, dex, run);
    // key = (vkey - spl[d+1]) << ib1 | (imax - idx) << 1 | negzero with
    // idx = view-row << logb | bucket, as one sum of its disjoint fields
    const uint32_t kb0 = 2u * (a.geo.imax - (uint32_t)(col0 + (int64_t)g * V));
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const uint32_t d = ST ? (rec[i] >> 10) & 31u : owner(rec[i], act);
      const uint32_t dd = d < (uint32_t)C ? d : 0u;  // in-range reads for unselected items
      const uint32_t pos = lsd::digit_base<NT>(cnt, dd) + (ST ? (rec[i] >> 5) & 31u : (rec[i] >> 11) & 31u);
      const uint32_t t = ST ? (rec[i] >> 1) & 15u : (rec[i] >> 1) & 0x3FFu;
      const uint32_t key = ((rec[i] >> 16) << ib1) - kofs[dd] + kb0 - 2u * (uint32_t)(i / KB) - (t << lb1) +
                           (rec[i] & 1u);
      if (d < (uint32_t)C && pos < capc) seg[dd * ostride + pos] = key;
    }
    __syncthreads();
    if (tid < C) run[tid] += sendcnt[tid];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
  if (lane == 0) atomicMax(&s_max, mx);
  if (__syncthreads_or(bad) && tid == 0 && a.flag) atomicOr(a.flag, 1u);
  uint32_t* cn = A.cnt + ((int64_t)rl * C + c) * (C + 1);
  if (tid < C) cn[tid] = run[tid];
  if (tid == C) cn[C] = s_max;
}

template <int DT>
__global__ void __launch_bounds__(XB_SNT, XB_SMIN) xb_sort(XBArgs A) {
  using KT = uint32_t;
  constexpr int NT = XB_SNT, NW = NT / 32, ITEMS = XB_ITEMS, C = XB_C;
  const XArgs& a = A.x;
  const int tid = threadIdx.x, lane = tid & 31;
  const int d = blockIdx.x, rl = blockIdx.y;
  const int64_t row = A.r0 + rl;
  const int ib1 = a.geo.ib + 1;
  extern __shared__ __align__(128) uint8_t xsm[];
  KT* buf = reinterpret_cast<KT*>(xsm);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(buf + padk<KT>(XB_CAP));
  __shared__ uint32_t ws[NW][8];
  __shared__ uint32_t dtot[16], dex[16];
  __shared__ uint32_t cn[C][C + 1];
  __shared__ uint32_t lspl[C + 1];
  __shared__ uint32_t tot[C], pre[C + 1];
  __shared__ uint32_t s_vary, s_and;
  __shared__ int s_why;
  __shared__ uint32_t s_start;
  pdl_trigger();
  pdl_wait();  // the partition launch produced the counts and sub-slots
  for (int i = tid; i < C * (C + 1); i += NT) cn[i / (C + 1)][i % (C + 1)] = A.cnt[(int64_t)rl * C * (C + 1) + i];
  if (tid <= C) lspl[tid] = A.spl[row * (C + 1) + tid];
  if (tid == 0) { s_vary = 0u; s_and = ~0u; }
  __syncthreads();
  if (tid < 32) {  // verdict and offsets, one warp (identical in every CTA of the row)
    const int q = lane;  // lanes < C: owner q (totals, checks); chunk q (this owner's prefix)
    uint32_t t = 0, over = 0;
    if (q < C) {
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const uint32_t v = cn[c][q];
        t += v;
        over |= v > (uint32_t)A.capc ? 1u : 0u;  // a sub-slot overflowed
      }
    }
    const uint32_t mx = __reduce_max_sync(0xFFFFFFFFu, q < C ? cn[q][C] : 0u);  // the row's max vkey
    uint32_t inc = t;  // inclusive prefix of the owner totals
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if (lane >= o) inc += v;
    }
    const uint32_t sum = __shfl_sync(0xFFFFFFFFu, inc, C - 1);
    const int tb = (int)lspl[0];
    uint32_t why = over;
    if (q < C) {
      if (t > (uint32_t)XB_CAP) why |= 1u;
      // the owner's value offsets must fit the 32-bit key above the index field
      const uint32_t hi = q == 0 ? mx : (lspl[q] - 1u) >> tb;
      if (t && ((uint64_t)(hi - (lspl[q + 1] >> tb)) >> (32 - ib1)) != 0ull) why |= 2u;
      tot[q] = t;
    }
    why = __reduce_or_sync(0xFFFFFFFFu, why);
    if (lspl[1] - lspl[C] > (uint32_t)LUTN) why |= 2u;
    if (sum < (uint64_t)a.k) why |= 4u;
    // this owner's sub-slot prefix over the chunks (lane = chunk)
    const uint32_t v = q < C ? cn[q][d] : 0u;
    uint32_t pinc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t w = __shfl_up_sync(0xFFFFFFFFu, pinc, o);
      if (lane >= o) pinc += w;
    }
    if (q <= C) pre[q] = pinc - v;  // lane C: the owner's total
    if (q == d) s_start = inc - t;
    if (lane == 0) {
      s_why = (int)why;
      if (why && d == 0) a.fb_list[atomicAdd(a.fb_count, 1)] = (int)row;
    }
  }
  __syncthreads();
  const int R = (int)tot[d];
  const int64_t start = s_start;
  if (s_why || R == 0 || start >= a.k) return;
  // ---- gather the C sub-slots in chunk order (bucket order within a
  // chunk) straight into registers, thread-blocked: position p = tid*items+i
  const int items = (R + NT - 1) / NT;
  KT key[ITEMS];
  {
    const uint32_t* seg = A.seg + ((int64_t)rl * C + d) * C * A.capc;
    const int p0 = tid * items;
    int cc = 0;  // sub-slot holding p0: the last with pre[cc] <= p0
#pragma unroll
    for (int st = C / 2; st > 0; st >>= 1)
      if (pre[cc + st] <= (uint32_t)p0) cc += st;
    KT kor = 0, kand = ~(KT)0;
    // addresses first (shared-memory walk over the chunk prefixes), then
    // every load at once: one global latency per thread, not one per key
    uint32_t off[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int p = p0 + i;
      off[i] = 0xFFFFFFFFu;
      if (i < items && p < R) {
        while (pre[cc + 1] <= (uint32_t)p) ++cc;
        off[i] = (uint32_t)cc * (uint32_t)A.capc + (uint32_t)(p - (int)pre[cc]);
      }
    }
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) key[i] = off[i] != 0xFFFFFFFFu ? seg[off[i]] : (KT)0;  // pads (0) sort last
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      if (off[i] != 0xFFFFFFFFu) {
        kor |= key[i];
        kand &= key[i];
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      kor |= __shfl_xor_sync(0xFFFFFFFFu, kor, o);
      kand &= __shfl_xor_sync(0xFFFFFFFFu, kand, o);
    }
    if (lane == 0) {
      atomicOr(&s_vary, (uint32_t)kor);
      atomicAnd(&s_and, (uint32_t)kand);
    }
  }
  __syncthreads();
  // ---- 4-bit LSD passes over the bits above the bucket id that vary (keys
  // in registers, one shared buffer); buf ends in sorted order
  const KT vary = s_vary ^ s_and;
  const int lowbit = 1 + a.logb;
  int shift = lowbit;
  if ((vary >> lowbit) != 0) shift = lowbit + __ffs((int)(vary >> lowbit)) - 1;
  bool none = true;
  for (; shift < 32 && (vary >> shift) != 0; shift += 4) {
    if (((vary >> shift) & (KT)0xF) == 0) continue;
    if (!none) {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i)
        if (i < items) key[i] = buf[padk<KT>(tid * items + i)];
    }
    none = false;
    // per item FB bits: digit << (FB - 4) | rank among the thread's items of that digit
    constexpr int FB = ITEMS <= 16 ? 8 : 10, RM = (1 << (FB - 4)) - 1;
    constexpr int SPW = 32 / FB, SLW = (ITEMS + SPW - 1) / SPW;
    uint32_t sl[SLW];
#pragma unroll
    for (int q = 0; q < SLW; ++q) sl[q] = 0u;
#pragma unroll
    for (int q = 0; q < 8; ++q) cnt[q * NT + tid] = 0u;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      if (i < items) {
        const uint32_t dg = 15u - (uint32_t)((key[i] >> shift) & (KT)0xF);
        sl[i / SPW] |= ((dg << (FB - 4)) | lsd::count_digit<NT>(cnt, dg)) << (FB * (i % SPW));
      }
    }
    lsd::digit_scan<NT, 8>(cnt, ws, dtot, dex);  // its barriers order every read of buf before the stores
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      if (i < items) {
        const uint32_t bf = (sl[i / SPW] >> (FB * (i % SPW))) & ((1u << FB) - 1u);
        const uint32_t dg = bf >> (FB - 4);
        const int r = (int)(dex[dg] + lsd::digit_base<NT>(cnt, dg) + (bf & (uint32_t)RM));
        buf[padk<KT>(r)] = key[i];
      }
    }
    __syncthreads();
  }
  if (none) {  // already in order
#pragma unroll
    for (int i = 0; i < ITEMS; ++i)
      if (i < items) buf[padk<KT>(tid * items + i)] = key[i];
    __syncthreads();
  }
  const KT* src = buf;
  const int keep = (int)min((int64_t)R, a.k - start);
  const uint32_t vbase = lspl[d + 1] >> (int)lspl[0];
  // 32-bit decode (16-bit dtypes, index field <= 26 bits): value bits from
  // the owner's base vkey plus the key's offset, index = imax - field
  const int64_t obase = row * a.k + start;
  for (int q = tid; q < keep; q += NT) {
    const KT key = src[padk<KT>(q)];
    const uint32_t vk = vbase + (key >> ib1);
    store_bits<DT>(a.out_vals, obase + q, bits_of_key<DT>(vk, key & 1u));
    a.out_idx[obase + q] = (int64_t)(a.geo.imax - ((key >> 1) & a.geo.imax));
  }
}

constexpr size_t XB_PART_SMEM = (size_t)8 * XB_NT * 4;
constexpr size_t XB_SORT_SMEM = (size_t)padk<uint32_t>(XB_CAP) * 4 + (size_t)8 * XB_SNT * 4;

// rows per batch: at most 148 (measured best of 32/64/148 on cfg5); the
// workspace is sized for the cap, BTK_XB_ROWS may only lower it
constexpr int XB_ROWS_CAP = 148;
inline int xb_rows_cap(int64_t m) { return (int)std::min<int64_t>(m, XB_ROWS_CAP); }
inline int xb_rows(int64_t m) {
  return std::min(xb_rows_cap(m), std::max(1, fz::env_int("BTK_XB_ROWS", XB_ROWS_CAP)));
}

template <int DT, int KB>
cudaError_t xb_attrs() {
  static thread_local int attr_done = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_done == dev) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute((const void*)xb_sort<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)XB_SORT_SMEM);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute((const void*)xb_part<DT, KB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)XB_PART_SMEM);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute((const void*)xb_part<DT, KB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)XB_PART_SMEM);
  if (e != cudaSuccess) return e;
  attr_done = dev;
  return cudaSuccess;
}

// Side stream for the owner sorts (per host thread and device): batch i's
// sort overlaps batch i+1's partition; the partition and sort buffers are
// double-buffered, so partition i+2 waits for sort i only.
struct XBSide {
  cudaStream_t s = nullptr;
  cudaEvent_t part[2] = {nullptr, nullptr}, sort[2] = {nullptr, nullptr}, fork = nullptr;
};
inline cudaError_t xb_side(XBSide*& out) {
  static thread_local std::unordered_map<int, XBSide> side;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  XBSide& x = side[dev];
  if (!x.s) {
    e = cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
      e = cudaEventCreateWithFlags(&x.part[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x.sort[i], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  out = &x;
  return cudaSuccess;
}
inline bool xb_two_streams() { return fz::env_int("BTK_XB_STREAMS", 1) != 0; }

template <int DT, int KB>
cudaError_t xb_launch_all(XBArgs A, cudaStream_t st) {
  cudaError_t e = xb_attrs<DT, KB>();
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cfg.stream = st;
  cfg.blockDim = dim3(XB_NT);
  cfg.gridDim = dim3((unsigned)A.x.m);
  e = cudaLaunchKernelEx(&cfg, xb_split<DT, KB>, A);
  if (e != cudaSuccess) return e;
  const int br = xb_rows(A.x.m);
  const int64_t nbatch = (A.x.m + br - 1) / br;
  XBSide* sd = nullptr;
  const bool two = xb_two_streams() && nbatch > 1;
  if (two) {
    e = xb_side(sd);
    if (e != cudaSuccess) return e;
    e = cudaEventRecord(sd->fork, st);  // the side stream joins st's work (and a capture) here
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sd->s, sd->fork, 0);
    if (e != cudaSuccess) return e;
  }
  uint32_t* seg0 = A.seg;
  uint32_t* cnt0 = A.cnt;
  for (int64_t i = 0; i < nbatch; ++i) {
    const int buf = two ? (int)(i & 1) : 0;
    A.r0 = i * br;
    A.br = (int)std::min<int64_t>(br, A.x.m - A.r0);
    A.seg = seg0 + (size_t)buf * A.seg_elems;
    A.cnt = cnt0 + (size_t)buf * A.cnt_elems;
    cfg.gridDim = dim3(XB_C, (unsigned)A.br);
    cfg.blockDim = dim3(XB_NT);
    cfg.dynamicSmemBytes = XB_PART_SMEM;
    cfg.stream = st;
    if (two && i >= 2) {
      e = cudaStreamWaitEvent(st, sd->sort[buf], 0);  // sort i-2 released this buffer
      if (e != cudaSuccess) return e;
    }
    e = A.x.s <= 16 ? cudaLaunchKernelEx(&cfg, xb_part<DT, KB, true>, A)
                    : cudaLaunchKernelEx(&cfg, xb_part<DT, KB, false>, A);
    if (e != cudaSuccess) return e;
    cfg.dynamicSmemBytes = XB_SORT_SMEM;
    cfg.blockDim = dim3(XB_SNT);
    if (two) {
      e = cudaEventRecord(sd->part[buf], st);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(sd->s, sd->part[buf], 0);
      if (e != cudaSuccess) return e;
      cfg.stream = sd->s;
      cfg.numAttrs = 0;  // fully ordered after its partition (event)
      e = cudaLaunchKernelEx(&cfg, xb_sort<DT>, A);
      cfg.numAttrs = pdl_enabled() ? 1 : 0;
      if (e == cudaSuccess) e = cudaEventRecord(sd->sort[buf], sd->s);
    } else {
      e = cudaLaunchKernelEx(&cfg, xb_sort<DT>, A);
    }
    if (e != cudaSuccess) return e;
  }
  if (two) {  // join: st continues after the last sorts
    for (int b = 0; b < 2; ++b) {
      e = cudaStreamWaitEvent(st, sd->sort[b], 0);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

// ================================================================ host side
template <int DT> struct Cfg;
template <> struct Cfg<F32> {
  using KT = uint64_t;
  static constexpr int C = 8, NT = 512, IPT = 8, ITEMS = 8;
};
template <> struct Cfg<BF16> {
  using KT = uint32_t;
  static constexpr int C = 16, NT = 512, IPT = 16, ITEMS = 16;
};
template <> struct Cfg<F16> : Cfg<BF16> {};

inline bool pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

template <int DT>
bool plan_t(const Problem& p, XArgs& a) {
  using CF = Cfg<DT>;
  constexpr int V = Vec<DT>::V;
  const int esz = VT<DT>::W / 8;
  if (p.layout != 0 || !(p.kb == 1 || p.kb == 2 || p.kb == 4 || (p.kb == 8 && DT == F32))) return false;
  if (V * p.kb > 32) return false;
  if (!pow2(p.b) || p.n % p.b) return false;
  const int64_t s = p.n / p.b;
  if (s < p.kb || s > 1024) return false;
  if ((reinterpret_cast<uintptr_t>(p.x) & 15) || ((p.row_stride * esz) & 15)) return false;
  if (p.b % ((int64_t)CF::C * V * 32)) return false;  // whole warps of vector columns per CTA
  const int64_t cols = p.b / CF::C;
  const int64_t ncand = cols * p.kb;
  if (ncand > (int64_t)CF::IPT * CF::NT || ncand < SPC) return false;
  // expected keys per owner (k/C plus the threshold margin) within ~half the receive capacity
  if ((p.k + CF::C - 1) / CF::C > (int64_t)CF::NT * CF::ITEMS / 2) return false;
  if (p.m * CF::C > 0x7FFFFFFFll) return false;
  if (DT != F32 && p.geo.ib > 26) return false;
  a.x = p.x; a.row_stride = p.row_stride;
  a.m = p.m; a.n = p.n; a.k = p.k; a.b = p.b;
  a.s = (int)s;
  a.logb = 0;
  while ((int64_t(1) << a.logb) < p.b) ++a.logb;
  a.cols = (int)cols;
  a.ncand = (int)ncand;
  a.geo = p.geo;
  a.flag = p.flag;
  return true;
}

template <int DT, int KB>
cudaError_t launch_t(const XArgs& a, cudaStream_t st) {
  using CF = Cfg<DT>;
  using KT = typename CF::KT;
  using L = Layout<KT, CF::NT, CF::IPT, CF::ITEMS>;
  auto kern = fused_xchg<DT, KB, CF::C, CF::NT, CF::IPT, CF::ITEMS, KT>;
  static thread_local int attr_done = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_done != dev) {
    cudaError_t e = cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)L::BYTES);
    if (e != cudaSuccess) return e;
    if (CF::C > 8) {
      e = cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    attr_done = dev;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(a.m * CF::C));
  cfg.blockDim = dim3(CF::NT);
  cfg.dynamicSmemBytes = L::BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  attr[na].id = cudaLaunchAttributeClusterDimension;
  attr[na].val.clusterDim.x = CF::C;
  attr[na].val.clusterDim.y = 1;
  attr[na].val.clusterDim.z = 1;
  ++na;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int DT>
cudaError_t launch_dt(const XArgs& a, int64_t kb, cudaStream_t st) {
  switch (kb) {
    case 1: return launch_t<DT, 1>(a, st);
    case 2: return launch_t<DT, 2>(a, st);
    case 4: return launch_t<DT, 4>(a, st);
  }
  if constexpr (DT == F32) return launch_t<DT, 8>(a, st);
  return cudaErrorNotSupported;
}

bool plan(const Problem& p, XArgs& a) {
  switch (p.dtype) {
    case F32: return plan_t<F32>(p, a);
    case BF16: return plan_t<BF16>(p, a);
    case F16: return plan_t<F16>(p, a);
  }
  return false;
}

}  // namespace xc

bool xchg_supported(const Problem& p) {
  const int want = fz::env_int("BTK_XC", -1);
  if (want == 0) return false;
  // 16-bit dtypes with pools beyond one CTA's shared memory (<= 16384: the
  // single-CTA fused kernels are faster; fp32: the chunked pool path, whose
  // 64-bit keys this kernel sorts slower — BTK_XC=1 forces it for A/B runs)
  if (want != 1 && (p.dtype == F32 || p.b * p.kb <= fz::FUSED_POOL_CAP)) return false;
  if (p.b * p.kb < 8192) return false;
  xc::XArgs a{};
  return xc::plan(p, a);
}

static size_t al256(size_t v) { return (v + 255) & ~(size_t)255; }

namespace xc {
// 16-bit dtypes run the batched pipeline (1.6x the cluster kernel on cfg5);
// BTK_XB=0 selects the cluster kernel (development A/B)
inline bool use_batched(const Problem& p) { return p.dtype != F32 && fz::env_int("BTK_XB", 1) != 0; }

inline int xb_capc(const Problem& p, int ncand) {
  // expected keys per (owner, chunk): the kept fraction of the chunk over C
  // owners; 2x plus a margin (owners vary by whole values and by the
  // sampling error of the splitters), rounded to whole 128-byte lines
  const double e = (double)xb_rthr(p.k, p.b * p.kb) / SPC * ncand / XB_C;
  const int c = ((int)(2.0 * e) + 128 + 31) & ~31;
  return std::min(c, XB_CAP);
}

struct XBBufs {
  size_t spl, seg, cnt, total;
};
inline XBBufs xb_bufs(const Problem& p) {
  const size_t br = (size_t)xb_rows_cap(p.m);
  const int ncand = (int)(p.b / XB_C * p.kb);
  XBBufs u{};
  u.spl = al256((size_t)p.m * (XB_C + 1) * 4);
  u.seg = 2 * al256(br * XB_C * XB_C * (size_t)xb_capc(p, ncand) * 4);  // double-buffered
  u.cnt = 2 * al256(br * XB_C * (XB_C + 1) * 4);
  u.total = u.spl + u.seg + u.cnt;
  return u;
}

template <int DT>
cudaError_t run_batched(const Problem& p, const XArgs& a, uint8_t* w, cudaStream_t st) {
  const XBBufs u = xb_bufs(p);
  XBArgs A{};
  A.x = a;
  A.capc = xb_capc(p, a.ncand);
  A.spl = reinterpret_cast<uint32_t*>(w);
  A.seg = reinterpret_cast<uint32_t*>(w + u.spl);
  A.cnt = reinterpret_cast<uint32_t*>(w + u.spl + u.seg);
  A.seg_elems = u.seg / 2 / 4;
  A.cnt_elems = u.cnt / 2 / 4;
  switch (p.kb) {
    case 1: return xb_launch_all<DT, 1>(A, st);
    case 2: return xb_launch_all<DT, 2>(A, st);
    case 4: return xb_launch_all<DT, 4>(A, st);
  }
  return cudaErrorNotSupported;
}
}  // namespace xc

int xchg_launch_count(const Problem& p) {
  if (!xc::use_batched(p)) return 2;
  const int64_t br = xc::xb_rows(p.m);
  return (int)(2 + 2 * ((p.m + br - 1) / br));
}

size_t xchg_workspace_bytes(const Problem& p) {
  // fallback-row counter + list, one scratch slot (pool + k keys) per
  // fallback CTA, and the batched pipeline's per-batch buffers
  const int64_t P = p.b * p.kb;
  const int64_t ctas = std::min<int64_t>(p.m, xc::FB_CTAS);
  // (sized whenever the batched pipeline may run, so the choice can change
  // between preparing a workspace and launching on it)
  const size_t xb = p.dtype != F32 ? xc::xb_bufs(p).total : 0;
  return al256(4) + al256((size_t)p.m * 4) + al256((size_t)ctas * (P + p.k) * 8) + xb;
}

cudaError_t run_xchg(const Problem& p, void* ws, void* out_vals, int64_t* out_idx, cudaStream_t st) {
  xc::XArgs a{};
  if (!xc::plan(p, a)) return cudaErrorNotSupported;
  uint8_t* w = static_cast<uint8_t*>(ws);
  int* count = reinterpret_cast<int*>(w);
  w += al256(4);
  int* list = reinterpret_cast<int*>(w);
  w += al256((size_t)p.m * 4);
  uint64_t* slots = reinterpret_cast<uint64_t*>(w);
  const int64_t P = p.b * p.kb;
  a.out_vals = out_vals;
  a.out_idx = out_idx;
  a.fb_count = count;
  a.fb_list = list;
  a.trace = fz::env_int("BTK_XC_TRACE", 0);
  a.early = (p.flags & 1u) && fz::pdl_enabled() ? 1 : 0;
  cudaError_t e = cudaMemsetAsync(count, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  const int64_t ctas = std::min<int64_t>(p.m, xc::FB_CTAS);
  uint8_t* xbw = reinterpret_cast<uint8_t*>(slots) + al256((size_t)ctas * (P + p.k) * 8);
  switch (xc::use_batched(p) ? -p.dtype - 1 : p.dtype) {
    case -BF16 - 1: e = xc::run_batched<BF16>(p, a, xbw, st); break;
    case -F16 - 1: e = xc::run_batched<F16>(p, a, xbw, st); break;
    case F32: e = xc::launch_dt<F32>(a, p.kb, st); break;
    case BF16: e = xc::launch_dt<BF16>(a, p.kb, st); break;
    case F16: e = xc::launch_dt<F16>(a, p.kb, st); break;
    default: e = cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  // rows the partition could not place: the persistent fallback kernel
  switch (p.dtype) {
    case F32: return xc::launch_fallback<F32>(a, p.kb, slots, P + p.k, st);
    case BF16: return xc::launch_fallback<BF16>(a, p.kb, slots, P + p.k, st);
    default: return xc::launch_fallback<F16>(a, p.kb, slots, P + p.k, st);
  }
}

}  // namespace btk

// Development timeline of the last traced fused_xchg launch (BTK_XC_TRACE=1):
// per CTA, globaltimer at start, stage 1 done, after barriers A, B (+ splitter
// copy), C, D, sort done, end.  Not part of the ABI.
extern "C" int btk_xc_trace_read(void* host_dst, int nblocks) {
  if (nblocks > btk::xc::TRACE_CTAS) nblocks = btk::xc::TRACE_CTAS;
  return (int)cudaMemcpyFromSymbol(host_dst, btk::xc::g_xtrace, (size_t)nblocks * 8 * 8);
}
