"""Adversarial inputs for the ordering contract: subnormals and signed zeros.

The reference orders by "value descending (IEEE compare: -0.0 == +0.0,
subnormals exact), then index ascending" and returns the input's own bits
(reference exact.py:130-139, approx.py:151-162).  These generators build
inputs whose k-th boundary falls INSIDE the subnormal / zero band, directly
as bit patterns of the target dtype, so every value is exactly
representable in it (bf16 subnormals: exponent field 0 of 8; fp16: exponent
field 0 of 5 — those are normal numbers in fp32, but subnormal for the
16-bit kernels' packed compares).

Returned as float32 arrays (exact upcasts) for the oracle; `to_dtype`
gives the device tensor with the intended bits.
"""

from __future__ import annotations

import numpy as np
import torch

# (sign bit, exponent field shift, mantissa bits, exponent bias) per dtype
_FMT = {"f32": (31, 23, 23), "bf16": (15, 7, 7), "f16": (15, 10, 10)}
TORCH = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}


def _pack(sign, exp, mant, dn):
    sb, es, _ = _FMT[dn]
    raw = (sign.astype(np.uint64) << sb) | (exp.astype(np.uint64) << es) | mant.astype(np.uint64)
    if dn == "f32":
        return raw.astype(np.uint32).view(np.float32)
    u16 = raw.astype(np.uint16)
    t = torch.from_numpy(u16.view(np.int16)).view(TORCH[dn])
    return t.float().numpy()


def special(rng: np.random.Generator, kind: str, m: int, n: int, dn: str) -> np.ndarray:
    """kind: 'subnormal' | 'pm0' | 'subnormal_ties'."""
    _, _, mb = _FMT[dn]
    shape = (m, n)
    u = rng.random(shape)
    sign = (rng.random(shape) < 0.5).astype(np.uint64)
    if kind == "pm0":
        # +-0 soup: the k-th boundary sits among equal zeros of both signs
        exp = np.zeros(shape, np.uint64)
        mant = np.zeros(shape, np.uint64)
        neg = u < 0.10                     # -1.0 (exponent = bias)
        one = (u >= 0.10) & (u < 0.103)    # +1.0 (rare: most bucket maxima are zeros)
        bias = {"f32": 127, "bf16": 127, "f16": 15}[dn]
        exp[neg | one] = bias
        sign[neg] = 1
        sign[one] = 0
        return _pack(sign, exp, mant, dn)
    # subnormal band: exponent field 0, non-zero mantissa; a few exact
    # zeros of both signs and a few tiny normals (exponent 1) on top
    if kind == "subnormal_ties":
        mant = rng.integers(1, 8, size=shape).astype(np.uint64)   # heavy ties
    else:
        mant = rng.integers(1, 1 << mb, size=shape).astype(np.uint64)
    exp = np.zeros(shape, np.uint64)
    zero = u < 0.15
    mant[zero] = 0
    tiny_normal = (u >= 0.15) & (u < 0.155)
    exp[tiny_normal] = 1
    big_neg = (u >= 0.155) & (u < 0.30)       # ordinary negatives below the band
    out = _pack(sign, exp, mant, dn)
    out[big_neg] = -1.0
    return out


def to_dtype(x32: np.ndarray, dn: str) -> torch.Tensor:
    """Exact: every value of `x32` is representable in `dn`."""
    t = torch.from_numpy(np.ascontiguousarray(x32)).to(TORCH[dn])
    assert torch.equal(t.float().view(torch.int32), torch.from_numpy(np.ascontiguousarray(x32)).view(torch.int32)), \
        "input not exactly representable (bits changed in the cast)"
    return t


def has_subnormal(x32: np.ndarray, dn: str) -> bool:
    a = np.abs(x32[x32 != 0])
    tiny = {"f32": np.float32(1.17549435e-38), "bf16": np.float32(1.17549435e-38),
            "f16": np.float32(6.1035156e-05)}[dn]
    return bool((a < tiny).any())
