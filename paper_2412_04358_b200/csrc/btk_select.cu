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
#include <cooperative_groups.h>

#include "btk_internal.h"
#include "btk_rank.cuh"
#include "btk_sort.cuh"

namespace btk {

namespace cg = cooperative_groups;

template <int DT>
__device__ __forceinline__ void emit(uint64_t c, int64_t pos, const CompGeo& g, void* out_vals,
                                     int64_t* out_idx) {
  uint32_t bits;
  int64_t idx;
  decode_comp<DT>(c, g, bits, idx);
  store_bits<DT>(out_vals, pos, bits);
  out_idx[pos] = idx;
}

// ---------------------------------------------------------------------------
// One CTA per segment of L <= NT*ITEMS keys: keys into shared memory, the
// bucketing/rank engine (btk_rank.cuh) finds the kk largest in order.
template <int DT, int NT, int ITEMS, bool DECODE>
__global__ void __launch_bounds__(NT) k2_small(const uint64_t* __restrict__ in, int64_t in_stride,
                                               int64_t L, int64_t kk, uint64_t* __restrict__ out_keys,
                                               void* __restrict__ out_vals,
                                               int64_t* __restrict__ out_idx, int64_t out_stride,
                                               CompGeo g, int lognb, const uint32_t* only) {
  if (only && only[blockIdx.x] == 0u) return;  // segment already done by k2_cluster
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint64_t* sk = reinterpret_cast<uint64_t*>(smem_raw);
  uint8_t* aux = smem_raw + ((size_t)L * 8 + 127) / 128 * 128;
  const RankSmem S = rank_smem(sk, aux, L, kk, lognb, NT);
  const int64_t seg = blockIdx.x;
  const uint64_t* src = in + seg * in_stride;
  for (int p = threadIdx.x; p < L; p += NT) sk[p] = src[p];
  __syncthreads();
  rank_select_sort<DT, NT, ITEMS>(S, (int)L, (int)kk, lognb, g.ib);
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

// ---------------------------------------------------------------------------
// Long segments (16384 < L <= 8 * 16384, e.g. cfg5: 131072 -> 65536): one
// thread-block CLUSTER of S CTAs per segment, the keys spread over the S
// shared memories, the bucketing/rank engine distributed through DSMEM:
//
//   1. CTA c loads keys [c*L/S, (c+1)*L/S) into registers; cluster-wide
//      min / max (DSMEM) fix ONE bucketing rule (btk_rank.cuh RsRule);
//   2. local bucket histograms with slots; every CTA reads all S histograms
//      -> global bucket starts and its own offset inside every bucket;
//   3. bucket d belongs to the CTA owning output position gstart[d]
//      (ranges of ceil(kk/S)); buckets starting at or beyond kk are dropped;
//      each key is stored straight into its owner's shared memory (DSMEM)
//      at its bucket-order position;
//   4. every CTA ranks its received buckets locally (rank engine, big
//      buckets refined recursively) and writes its contiguous slice of the
//      output, coalesced.
//
// If a CTA would receive more keys than it can hold (adversarially skewed
// buckets), the segment is flagged in seg_fail and left to the radix-select
// + LSD fallback launched after this kernel (which skips unflagged
// segments), so correctness never depends on the value distribution.
__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

constexpr int KC_NT = 512, KC_ITEMS = 32, KC_CAP = KC_NT * KC_ITEMS, KC_LOGNB = 11;
constexpr int KC_WLOGNB = 5;  // per-warp buckets when a warp ranks one big bucket

__host__ __device__ constexpr size_t kc_smem_bytes() {
  return (size_t)KC_CAP * 8 +                                   // pool / receive buffer
         (((size_t)(1 << KC_LOGNB) + 2) * 4 + 127) / 128 * 128 * 2 +  // gstart, gbase
         rank_aux_bytes(KC_NT, KC_LOGNB, KC_CAP, KC_CAP) + 256;
}

template <int DT>
__global__ void __launch_bounds__(KC_NT, 1) k2_cluster(const uint64_t* __restrict__ in,
                                                       int64_t in_stride, int64_t L, int64_t kk,
                                                       void* __restrict__ out_vals,
                                                       int64_t* __restrict__ out_idx,
                                                       int64_t out_stride, CompGeo g,
                                                       uint32_t* __restrict__ seg_fail) {
  constexpr int NB = 1 << KC_LOGNB;
  constexpr int NW = KC_NT / 32;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __shared__ uint64_t s_mm[2];
  __shared__ float s_vm[2];
  __shared__ int s_owner_base[9];
  __shared__ int s_fail;
  __shared__ int2 s_over[KC_CAP / (32 * KC_ITEMS) + 1];
  __shared__ int s_nover;
  __shared__ int s_lastkept;
  cg::cluster_group cluster = cg::this_cluster();
  const int S = (int)cluster.num_blocks();
  const int c = (int)cluster.block_rank();
  const int64_t seg = blockIdx.x / S;
  const int tid = threadIdx.x;
  uint64_t* pool = reinterpret_cast<uint64_t*>(smem_raw);
  uint32_t* gstart = reinterpret_cast<uint32_t*>(smem_raw + (size_t)KC_CAP * 8);
  uint32_t* gbase = gstart + (((size_t)NB + 2) * 4 + 127) / 128 * 32;
  uint8_t* aux = reinterpret_cast<uint8_t*>(gbase + (((size_t)NB + 2) * 4 + 127) / 128 * 32);
  const RankSmem R = rank_smem(pool, aux, KC_CAP, KC_CAP, KC_LOGNB, KC_NT);
  uint32_t* hist = R.hist;  // local bucket counts (read remotely in step 2)

  // ---- 1. keys -> registers, cluster-wide min / max
  const int64_t lo = (L * c) / S, hi = (L * (c + 1)) / S;
  const int n = (int)(hi - lo);
  const uint64_t* src = in + seg * in_stride + lo;
  uint64_t key[KC_ITEMS];
  uint32_t sd[KC_ITEMS];  // slot << 16 | bucket
  uint64_t mn = ~0ull, mx = 0ull;
  float vmn = __int_as_float(0x7F800000), vmx = -__int_as_float(0x7F800000);
#pragma unroll
  for (int i = 0; i < KC_ITEMS; ++i) {
    const int p = tid + i * KC_NT;
    key[i] = p < n ? __ldcs(src + p) : 0ull;
    if (key[i]) {
      mn = key[i] < mn ? key[i] : mn;
      mx = key[i] > mx ? key[i] : mx;
      const float v = comp_value<DT>(key[i], g.ib);
      vmn = fminf(vmn, v);
      vmx = fmaxf(vmx, v);
    }
  }
  for (int j = tid; j < NB + 2; j += KC_NT) hist[j] = 0u;
  block_minmax<KC_NT>(mn, mx, vmn, vmx, R.red);
  if (tid == 0) { s_mm[0] = mn; s_mm[1] = mx; s_vm[0] = vmn; s_vm[1] = vmx; s_fail = 0; s_nover = 0; }
  cluster.sync();
  for (int r = 0; r < S; ++r) {
    const uint64_t* rm = cluster.map_shared_rank(s_mm, r);
    const float* rv = cluster.map_shared_rank(s_vm, r);
    const uint64_t a0 = rm[0], a1 = rm[1];
    const float b0 = rv[0], b1 = rv[1];
    mn = a0 < mn ? a0 : mn;
    mx = a1 > mx ? a1 : mx;
    vmn = fminf(vmn, b0);
    vmx = fmaxf(vmx, b1);
  }
  RsRule rule;
  rule.nb = NB;
  rule.mn = mn;
  rule.vmx = vmx;
  rule.same = (mn == mx);
  rule.shift = max(0, bits64(mx - mn) - KC_LOGNB);
  const float span = vmx - vmn;
  rule.scale = (float)NB / span;
  const bool narrow_band = (vmn > 0.f && vmx < 4.f * vmn) || (vmx < 0.f && vmn > 4.f * vmx);
  rule.vmode = !narrow_band && (span > 0.f) && (rule.scale > 0.f) && (rule.scale < 3.0e38f) &&
               (span < 3.0e38f);
  if (rule.same) rule.vmode = false;  // identical keys: key mode puts them in one bucket

  // ---- 2. local histogram, then global bucket starts / my offsets
#pragma unroll
  for (int i = 0; i < KC_ITEMS; ++i) {
    if (tid + i * KC_NT < n) {
      const uint32_t d = (uint32_t)rs_bucket<DT>(rule, key[i], g.ib);
      sd[i] = (atomicAdd(&hist[d], 1u) << 16) | d;
    }
  }
  cluster.sync();  // all histograms complete
  for (int d = tid; d < NB + 2; d += KC_NT) {
    uint32_t tot = 0, before = 0;
    for (int r = 0; r < S; ++r) {
      const uint32_t v = cluster.map_shared_rank(hist, r)[d];
      before += (r < c) ? v : 0u;
      tot += v;
    }
    gstart[d] = tot;
    gbase[d] = before;
  }
  cluster.sync();  // remote histogram reads done: hist is free again
  block_exscan<KC_NT>(gstart, NB + 2, reinterpret_cast<uint32_t*>(R.red));
  for (int d = tid; d < NB + 2; d += KC_NT) gbase[d] += gstart[d];
  // owners: CTA o owns buckets whose start lies in [o*RR, (o+1)*RR)
  const int64_t RR = (kk + S - 1) / S;
  if (tid < 9) s_owner_base[tid] = -1;
  if (tid == 0) s_lastkept = -1;
  __syncthreads();
  for (int d = tid; d < NB; d += KC_NT) {
    const uint32_t st0 = gstart[d];
    if (gstart[d + 1] == st0 || (int64_t)st0 >= kk) continue;  // empty or dropped
    const int o = (int)imin64(S - 1, (int64_t)st0 / RR);
    atomicMin(reinterpret_cast<unsigned*>(&s_owner_base[o]), st0);  // -1 = 0xFFFFFFFF
    atomicMax(&s_lastkept, d);
  }
  __syncthreads();
  // kept keys end with the last bucket that starts below kk
  const int kept_end = s_lastkept >= 0 ? (int)gstart[s_lastkept + 1] : 0;
  // receive count of every owner must fit its buffer; identical in all CTAs
  if (tid < S) {
    const int o = tid;
    const int b0 = s_owner_base[o];
    if (b0 >= 0) {
      int end = kept_end;
      for (int o2 = o + 1; o2 < S; ++o2)
        if (s_owner_base[o2] >= 0) { end = s_owner_base[o2]; break; }
      if (end - b0 > KC_CAP) atomicOr(reinterpret_cast<unsigned*>(&s_fail), 1u);
    }
  }
  __syncthreads();
  if (s_fail) {
    if (c == 0 && tid == 0) seg_fail[seg] = 1u;
    return;  // uniform across the cluster (same data in every CTA)
  }
  if (c == 0 && tid == 0) seg_fail[seg] = 0u;

  // ---- 3. send every kept key to its owner's buffer (in bucket order)
#pragma unroll
  for (int i = 0; i < KC_ITEMS; ++i) {
    if (tid + i * KC_NT < n && key[i]) {
      const uint32_t d = sd[i] & 0xFFFFu;
      const uint32_t st0 = gstart[d];
      if ((int64_t)st0 >= kk) continue;
      const int o = (int)imin64(S - 1, (int64_t)st0 / RR);
      const int pos = (int)(gbase[d] + (sd[i] >> 16)) - s_owner_base[o];
      cluster.map_shared_rank(pool, o)[pos] = key[i];
      cluster.map_shared_rank(R.bid, o)[pos] = (uint16_t)d;
    }
  }
  cluster.sync();  // all keys delivered

  // ---- 4. rank the received buckets locally, emit my output slice
  const int base = s_owner_base[c];
  if (base < 0) return;  // owns nothing
  int nxt = -1;
  for (int o2 = c + 1; o2 < S; ++o2)
    if (s_owner_base[o2] >= 0) { nxt = s_owner_base[o2]; break; }
  const int cnt = (nxt >= 0 ? nxt : kept_end) - base;
  const int kloc = (int)imin64(cnt, kk - base);  // outputs this CTA writes
  for (int q = tid; q < kloc; q += KC_NT) R.inv[q] = RS_NONE;
  if (tid == 0) { R.ctl[0] = 0; R.ctl[1] = 0; }
  __syncthreads();
  for (int p = tid; p < cnt; p += KC_NT) {
    const uint64_t x = pool[p];
    const int d = R.bid[p];
    const int s0 = (int)gstart[d] - base, s1 = (int)gstart[d + 1] - base;
    if (s0 >= kloc) continue;
    if (rule.same) {
      if (p < kloc) R.inv[p] = (uint16_t)p;
      continue;
    }
    if (s1 - s0 > RS_LIMIT) {
      if (p == s0) {
        const int t = atomicAdd(&R.ctl[1], 1);
        R.work[t % RS_WORK] = make_int2(s0, s1);
      }
      continue;
    }
    int cntg = 0;
    for (int j = s0; j < s1; ++j) {
      const uint64_t y = pool[j];
      cntg += (y > x || (y == x && j < p)) ? 1 : 0;
    }
    const int f = s0 + cntg;
    if (f < kloc) R.inv[f] = (uint16_t)p;
  }
  __syncthreads();
  // Big buckets (typically one bf16 value shared by hundreds of indices):
  // one WARP each, in parallel (gbase is free scratch now); the rare ones
  // too large for a warp go through the CTA engine afterwards.
  {
    const int nbig = R.ctl[1];
    const int warp = tid >> 5;
    uint32_t* whist = gbase + warp * ((1 << KC_WLOGNB) + 2);
    for (int w = warp; w < nbig; w += NW) {
      const int2 r = R.work[w];
      const int sz = r.y - r.x;
      if (sz > 32 * KC_ITEMS) {
        if ((tid & 31) == 0) s_over[atomicAdd(&s_nover, 1)] = r;  // <= KC_CAP/1024 of them
        continue;
      }
      warp_rank_sort<DT, KC_ITEMS>(pool + r.x, sz, kloc - r.x, R.inv + r.x, R.bid + r.x, whist,
                                   KC_WLOGNB, g.ib, r.x);
    }
    __syncthreads();
    const int nover = s_nover;
    for (int w = 0; w < nover; ++w) {
      const int2 r = s_over[w];
      __syncthreads();
      if (tid == 0) { R.ctl[0] = 0; R.ctl[1] = 0; }
      __syncthreads();
      rs_range<DT, KC_NT, KC_ITEMS>(R, r.x, r.y, kloc, KC_LOGNB, g.ib);
      for (;;) {  // its own big buckets
        const int head = R.ctl[0], tail = R.ctl[1];
        if (head >= tail) break;
        const int2 r2 = R.work[head % RS_WORK];
        __syncthreads();
        if (tid == 0) R.ctl[0] = head + 1;
        rs_range<DT, KC_NT, KC_ITEMS>(R, r2.x, r2.y, kloc, KC_LOGNB, g.ib);
      }
    }
  }
  __syncthreads();
  for (int q = tid; q < kloc; q += KC_NT)
    emit<DT>(rs_key(pool, R.inv[q]), seg * out_stride + base + q, g, out_vals, out_idx);
}

// ---------------------------------------------------------------------------
// MSD radix select + compaction for one long segment per CTA.
template <int NT>
__global__ void __launch_bounds__(NT) k2_select_compact(const uint64_t* __restrict__ in,
                                                        int64_t in_stride, int64_t L, int64_t kk,
                                                        uint64_t* __restrict__ out,
                                                        int64_t out_stride, int nbits,
                                                        const uint32_t* only) {
  if (only && only[blockIdx.x] == 0u) return;
  __shared__ uint32_t hist[RADIX];
  __shared__ int s_bin;
  __shared__ uint32_t s_above;
  __shared__ uint32_t s_cnt;
  const int64_t seg = blockIdx.x;
  const uint64_t* src = in + seg * in_stride;
  uint64_t* dst = out + seg * out_stride;
  uint64_t prefix = 0;
  uint32_t need = (uint32_t)kk;
  int shift = nbits;
  bool early = false;
  while (shift > 0) {
    const int w = (shift % 8) ? (shift % 8) : 8;
    shift -= w;
    for (int j = threadIdx.x; j < RADIX; j += NT) hist[j] = 0;
    __syncthreads();
    const int hs = shift + w;
    for (int64_t p = threadIdx.x; p < L; p += NT) {
      uint64_t key = src[p];
      uint64_t hi = (hs >= 64) ? 0ull : (key >> hs);
      if (hi == prefix) atomicAdd(&hist[(uint32_t)(key >> shift) & ((1u << w) - 1u)], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) find_crossing_desc(hist, need, &s_bin, &s_above);
    __syncthreads();
    const int bin = s_bin;
    need -= s_above;
    prefix = (prefix << w) | (uint64_t)bin;
    const uint32_t inbin = hist[bin];
    __syncthreads();
    if (inbin == need) { early = true; break; }
  }
  // early: selected = {key >= prefix << shift}, exactly kk of them.
  // else : thr = prefix is an exact key value; {key > thr} has kk - need
  //        members, remaining slots are copies of thr (only the empty
  //        sentinel 0 can repeat).
  const uint64_t thr = early ? (prefix << shift) : prefix;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int64_t p0 = 0; p0 < L; p0 += NT) {
    int64_t p = p0 + threadIdx.x;
    uint64_t key = (p < L) ? src[p] : 0ull;
    bool take = (p < L) && (early ? (key >= thr) : (key > thr));
    uint32_t ball = __ballot_sync(0xFFFFFFFFu, take);
    uint32_t base = 0;
    if (lane == 0 && ball) base = atomicAdd(&s_cnt, (uint32_t)__popc(ball));
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    if (take) dst[base + __popc(ball & lanemask_lt())] = key;
  }
  __syncthreads();
  for (int64_t p = s_cnt + threadIdx.x; p < kk; p += NT) dst[p] = thr;
}

// ---------------------------------------------------------------------------
// Stable LSD sort of kk keys per segment through a global ping-pong buffer,
// one CTA per segment; the epilogue writes the sorted keys out.
template <int DT, int NT, int ITEMS, bool DECODE>
__global__ void __launch_bounds__(NT) k2_global_lsd(uint64_t* __restrict__ A, uint64_t* __restrict__ B,
                                                    int64_t stride, int64_t kk,
                                                    uint64_t* __restrict__ out_keys,
                                                    void* __restrict__ out_vals,
                                                    int64_t* __restrict__ out_idx,
                                                    int64_t out_stride, CompGeo g,
                                                    const uint32_t* only) {
  if (only && only[blockIdx.x] == 0u) return;
  constexpr int N = NT * ITEMS;
  constexpr int NW = NT / 32;
  __shared__ uint32_t whist[NW * RADIX];
  __shared__ uint32_t dtotal[RADIX];
  __shared__ uint32_t runbase[RADIX];
  __shared__ uint32_t ghist[RADIX];
  __shared__ int s_skip;
  const int64_t seg = blockIdx.x;
  uint64_t* src = A + seg * stride;
  uint64_t* dst = B + seg * stride;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int shift = 1; shift < g.nbits; shift += 8) {
    for (int j = threadIdx.x; j < RADIX; j += NT) ghist[j] = 0;
    if (threadIdx.x == 0) s_skip = 0;
    __syncthreads();
    for (int64_t p = threadIdx.x; p < kk; p += NT) atomicAdd(&ghist[desc_digit(src[p], shift)], 1u);
    __syncthreads();
    if (threadIdx.x < RADIX && ghist[threadIdx.x] == (uint32_t)kk) s_skip = 1;
    if (warp == 0) warp_exscan256(ghist, runbase);
    __syncthreads();
    if (s_skip) continue;
    for (int64_t t0 = 0; t0 < kk; t0 += N) {
      uint64_t key[ITEMS];
      uint32_t rank[ITEMS];
      bool valid[ITEMS];
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        int64_t p = t0 + warp * 32 * ITEMS + i * 32 + lane;
        valid[i] = p < kk;
        key[i] = valid[i] ? src[p] : 0ull;  // invalid tail ranks last (digit 255)
      }
      uint32_t* wh = whist + warp * RADIX;
      for (int j = lane; j < RADIX; j += 32) wh[j] = 0;
      __syncwarp();
      warp_rank<ITEMS>(key, shift, wh, rank);
      __syncthreads();
      warp_offsets<NT>(whist, dtotal);
      __syncthreads();
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        if (valid[i]) {
          uint32_t d = desc_digit(key[i], shift);
          dst[runbase[d] + whist[warp * RADIX + d] + rank[i]] = key[i];
        }
      }
      __syncthreads();
      for (int j = threadIdx.x; j < RADIX; j += NT) runbase[j] += dtotal[j];
      __syncthreads();
    }
    uint64_t* t = src; src = dst; dst = t;
  }
  __syncthreads();
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
static cudaError_t launch_small(const K2Args& a, cudaStream_t st, const uint32_t* only = nullptr) {
  auto kern = k2_small<DT, NT, ITEMS, DECODE>;
  const int lognb = rank_lognb(a.L);
  const size_t sm = ((size_t)a.L * 8 + 127) / 128 * 128 + rank_aux_bytes(NT, lognb, a.kk, a.L);
  cudaError_t e = ensure_smem_attr((const void*)kern, sm);
  if (e != cudaSuccess) return e;
  if (a.nseg == 0) return cudaSuccess;
  kern<<<(unsigned)a.nseg, NT, sm, st>>>(a.in, a.in_stride, a.L, a.kk, a.out_keys, a.out_vals,
                                         a.out_idx, a.out_stride, a.geo, lognb, only);
  return cudaGetLastError();
}

template <int DT, bool DECODE>
static cudaError_t run_small(const K2Args& a, cudaStream_t st, const uint32_t* only = nullptr) {
  const int64_t L = a.L;
  if (L <= 64) return launch_small<DT, 64, 1, DECODE>(a, st, only);
  if (L <= 256) return launch_small<DT, 128, 2, DECODE>(a, st, only);
  if (L <= 1024) return launch_small<DT, 256, 4, DECODE>(a, st, only);
  if (L <= 4096) return launch_small<DT, 512, 8, DECODE>(a, st, only);
  return launch_small<DT, 512, 32, DECODE>(a, st, only);
}

template <int DT>
static cudaError_t launch_cluster(const K2Args& a, cudaStream_t st) {
  const int S = (int)((a.L + KC_CAP - 1) / KC_CAP);
  auto kern = k2_cluster<DT>;
  const size_t sm = kc_smem_bytes();
  cudaError_t e = ensure_smem_attr((const void*)kern, sm);
  if (e != cudaSuccess) return e;
  if (S > 8) {
    e = cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(a.nseg * S));
  cfg.blockDim = dim3(KC_NT);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a.in, a.in_stride, a.L, a.kk, a.out_vals, a.out_idx,
                            a.out_stride, a.geo, a.seg_flag);
}

template <int DT, bool DECODE>
static cudaError_t run_k2_t(const K2Args& a, cudaStream_t st) {
  if (a.L <= K2_SMALL_CAP) return run_small<DT, DECODE>(a, st);
  // long segments
  if (a.scratch_a == nullptr || a.scratch_b == nullptr) return cudaErrorInvalidValue;
  const uint32_t* only = nullptr;
  if constexpr (DECODE) {
    if (a.seg_flag && a.L <= 8 * (int64_t)KC_CAP) {
      cudaError_t e = launch_cluster<DT>(a, st);
      if (e != cudaSuccess) return e;
      only = a.seg_flag;  // the fallback below runs only for flagged segments
    }
  }
  k2_select_compact<1024><<<(unsigned)a.nseg, 1024, 0, st>>>(a.in, a.in_stride, a.L, a.kk,
                                                             a.scratch_a, a.kk, a.geo.nbits, only);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (a.kk <= K2_SMALL_CAP) {
    K2Args b = a;
    b.in = a.scratch_a;
    b.in_stride = a.kk;
    b.L = a.kk;
    return run_small<DT, DECODE>(b, st, only);
  }
  k2_global_lsd<DT, 512, 8, DECODE><<<(unsigned)a.nseg, 512, 0, st>>>(
      a.scratch_a, a.scratch_b, a.kk, a.kk, a.out_keys, a.out_vals, a.out_idx, a.out_stride, a.geo,
      only);
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
