// Shared device helpers for the bucketed top-k kernels (sm_100a).
//
// Ordering contract (reference exact.py:130-139, approx.py:142-164): rows are
// selected and emitted by "value descending (IEEE compare: -0.0 == +0.0,
// subnormals exact), then original index ascending"; emitted values are the
// input's bits (sign of zero kept).
//
// Every score becomes a unique unsigned 64-bit "composite key" whose unsigned
// order IS that total order:
//
//     comp = vkey << (IB + 1) | (IMAX - idx) << 1 | negzero
//
//   vkey    order-preserving integer image of the value with -0 folded to +0
//           (W = 32 bits for fp32, 16 for bf16/fp16);
//   IB      bits needed for idx (IMAX = 2^IB - 1 >= n - 1), so a larger
//           comp has the smaller index among equal values;
//   negzero 1 iff the element was -0.0: never changes the order (comps are
//           unique without it) but lets the decoder restore the exact bits.
//
// comp == 0 is the "empty slot" sentinel: every finite value has vkey > 0.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace btk {

enum Dtype : int { F32 = 0, BF16 = 1, F16 = 2 };

template <int DT> struct VT;

template <> struct VT<F32> {
  using Bits = uint32_t;
  static constexpr int W = 32;
  static constexpr uint32_t SIGN = 0x80000000u;
  static constexpr uint32_t EXP = 0x7F800000u;
};
template <> struct VT<BF16> {
  using Bits = uint16_t;
  static constexpr int W = 16;
  static constexpr uint32_t SIGN = 0x8000u;
  static constexpr uint32_t EXP = 0x7F80u;
};
template <> struct VT<F16> {
  using Bits = uint16_t;
  static constexpr int W = 16;
  static constexpr uint32_t SIGN = 0x8000u;
  static constexpr uint32_t EXP = 0x7C00u;
};

// Order-preserving key of raw bits (held in a uint32).  -0 and +0 map to the
// same key.  Integer-only: no FTZ hazard for subnormals.
template <int DT>
__host__ __device__ __forceinline__ uint32_t vkey(uint32_t bits) {
  constexpr uint32_t S = VT<DT>::SIGN;
  constexpr uint32_t MASK = (VT<DT>::W == 32) ? 0xFFFFFFFFu : 0xFFFFu;
  bits = (bits == S) ? 0u : bits;
  return (bits & S) ? (~bits & MASK) : (bits | S);
}

template <int DT>
__host__ __device__ __forceinline__ uint32_t bits_of_key(uint32_t key, uint32_t negzero) {
  constexpr uint32_t S = VT<DT>::SIGN;
  constexpr uint32_t MASK = (VT<DT>::W == 32) ? 0xFFFFFFFFu : 0xFFFFu;
  if (negzero) return S;
  return (key & S) ? (key ^ S) : (~key & MASK);
}

template <int DT>
__host__ __device__ __forceinline__ bool nonfinite(uint32_t bits) {
  return (bits & VT<DT>::EXP) == VT<DT>::EXP;
}

template <int DT>
__host__ __device__ __forceinline__ uint32_t is_negzero(uint32_t bits) {
  return bits == VT<DT>::SIGN ? 1u : 0u;
}

// Composite-key geometry for one problem.
struct CompGeo {
  int ib;         // index bits
  uint32_t imax;  // 2^ib - 1
  int nbits;      // significant bits of a comp: W + ib + 1
};

__host__ __device__ __forceinline__ int bits_for(uint64_t v) {  // bits to hold v (0 -> 0)
  int b = 0;
  while (v) { ++b; v >>= 1; }
  return b;
}

template <int DT>
__host__ __device__ __forceinline__ CompGeo make_geo(int64_t n_or_label_space) {
  CompGeo g;
  g.ib = bits_for((uint64_t)(n_or_label_space - 1));
  g.imax = (g.ib >= 32) ? 0xFFFFFFFFu : ((1u << g.ib) - 1u);
  g.nbits = VT<DT>::W + g.ib + 1;
  return g;
}

__host__ __device__ __forceinline__ uint64_t make_comp(uint32_t key, uint32_t idx, uint32_t negz,
                                                        const CompGeo& g) {
  return ((uint64_t)key << (g.ib + 1)) | ((uint64_t)(g.imax - idx) << 1) | (uint64_t)negz;
}

template <int DT>
__host__ __device__ __forceinline__ void decode_comp(uint64_t c, const CompGeo& g, uint32_t& bits,
                                                     int64_t& idx) {
  uint32_t key = (uint32_t)(c >> (g.ib + 1));
  uint32_t field = (uint32_t)((c >> 1) & (uint64_t)g.imax);
  idx = (int64_t)(g.imax - field);
  bits = bits_of_key<DT>(key, (uint32_t)(c & 1));
}

// Raw element load (bits) for each dtype.
template <int DT>
__device__ __forceinline__ uint32_t load_bits(const void* base, int64_t off) {
  if constexpr (VT<DT>::W == 32) {
    return __ldg(reinterpret_cast<const uint32_t*>(base) + off);
  } else {
    return (uint32_t)__ldg(reinterpret_cast<const unsigned short*>(base) + off);
  }
}

template <int DT>
__device__ __forceinline__ void store_bits(void* base, int64_t off, uint32_t bits) {
  if constexpr (VT<DT>::W == 32) {
    reinterpret_cast<uint32_t*>(base)[off] = bits;
  } else {
    reinterpret_cast<unsigned short*>(base)[off] = (unsigned short)bits;
  }
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

}  // namespace btk
