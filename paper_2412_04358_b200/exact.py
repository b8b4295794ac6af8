"""Exact canonical selection on the GPU.

Mirrors reference `exact.py` (same public names):

* ``TopKResult`` / ``ScoredIndex``      -> exact.py:40-84
* ``exact_topk_oracle``                 -> exact.py:162-173 (full stable sort
  semantics; here a radix select + sort over composite keys)
* ``priority_queue_topk``               -> exact.py:176-220 (identical output
  by contract; same kernel)
* ``topk_with_indices``                 -> exact.py:142-159 (carried labels)

Results are canonical: value descending, ties by index (label) ascending,
values bit-identical to the selected inputs.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterator, List, NamedTuple

import numpy as np
import torch

from . import _lib, _ops
from .core import ConfigError

__all__ = ["ScoredIndex", "TopKResult", "exact_topk_oracle", "priority_queue_topk",
           "topk_with_indices"]


class ScoredIndex(NamedTuple):
    value: float
    index: int


@dataclass(frozen=True, eq=False)
class TopKResult:
    """(m, k) values (input dtype) and int64 indices, canonical per row."""

    values: torch.Tensor
    indices: torch.Tensor

    def __post_init__(self):
        if tuple(self.values.shape) != tuple(self.indices.shape) or self.values.ndim < 1:
            raise ValueError("values and indices must be matching arrays")

    @property
    def m(self) -> int:
        return self.values.shape[0]

    @property
    def k(self) -> int:
        return self.values.shape[-1]

    def row(self, r: int) -> List[ScoredIndex]:
        v = self.values[r].float().tolist()
        i = self.indices[r].tolist()
        return [ScoredIndex(float(a), int(b)) for a, b in zip(v, i)]

    def __iter__(self) -> Iterator[List[ScoredIndex]]:
        return (self.row(r) for r in range(self.m))

    def __eq__(self, other) -> bool:
        if not isinstance(other, TopKResult):
            return NotImplemented
        return (tuple(self.values.shape) == tuple(other.values.shape)
                and torch.equal(self.values.cpu(), other.values.cpu())
                and torch.equal(self.indices.cpu(), other.indices.cpu()))

    def numpy(self):
        return self.values.float().cpu().numpy(), self.indices.cpu().numpy()


def _check_k(k, n):
    # reference exact.py:99-103 (_check_k)
    if not isinstance(k, (int, np.integer)) or k < 1:
        raise ConfigError("nonpositive", f"k must be a positive integer, got {k!r}")
    if k > n:
        raise ConfigError("k_gt_n", f"k > n (k={k}, n={n})")


def _restore(t: torch.Tensor, lead, dim, orig_ndim):
    if orig_ndim <= 2 and (orig_ndim == 1 or dim % orig_ndim == orig_ndim - 1):
        return t
    t = t.reshape(*lead, t.shape[-1])
    return t.movedim(-1, dim % orig_ndim)


def exact_topk_oracle(scores, k: int, workers: int = 1, *, dim: int = -1,
                      check_finite: bool = True) -> TopKResult:
    """Exact canonical top-k per row (GPU).  ``workers`` is accepted for
    signature compatibility; the output never depends on it."""
    del workers
    t = _ops.to_device_tensor(scores)
    orig_ndim = t.ndim
    x, lead = _ops.as_rows(t, dim)
    m, n = x.shape
    _check_k(k, n)
    lib = _lib.load()
    dt = _ops.dtype_code(x)
    dev = x.device
    with torch.cuda.device(dev):
        vals = torch.empty((m, k), dtype=x.dtype, device=dev)
        idx = torch.empty((m, k), dtype=torch.int64, device=dev)
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
        wsb = lib.btk_exact_workspace_bytes(m, n, k, dt)
        ws = _ops.workspace(wsb, dev)
        st = lib.btk_exact_topk(x.data_ptr(), x.stride(0), dt, m, n, k, vals.data_ptr(),
                                idx.data_ptr(), ws.data_ptr(), wsb, flag.data_ptr(),
                                _ops.stream_handle(dev))
        _ops.raise_status(st, "(exact_topk)")
        if check_finite:
            _ops.check_flag(flag)
    return TopKResult(values=_restore(vals, lead, dim, orig_ndim),
                      indices=_restore(idx, lead, dim, orig_ndim))


def priority_queue_topk(scores, k: int, workers: int = 1, **kw) -> TopKResult:
    """Same contract as exact_topk_oracle (reference exact.py:195-220)."""
    return exact_topk_oracle(scores, k, workers, **kw)


def topk_with_indices(values, indices, k: int, *, check_finite: bool = True) -> TopKResult:
    """Canonical top-k of (value, carried label) pairs (reference exact.py:142-159).

    Labels must lie in [0, 2**31 - 1] (GPU composite-key width)."""
    v = _ops.to_device_tensor(values)
    i = torch.as_tensor(indices)
    if v.ndim == 1:
        v, i = v.unsqueeze(0), i.reshape(1, -1)
    if tuple(v.shape) != tuple(i.shape):
        raise ValueError("values and indices must have matching shapes")
    if v.ndim != 2:
        raise ValueError("values and indices must be (m, c) arrays")
    m, c = v.shape
    _check_k(k, c)
    v = v.contiguous()
    i = i.to(device=v.device, dtype=torch.int64).contiguous()
    lib = _lib.load()
    dt = _ops.dtype_code(v)
    dev = v.device
    with torch.cuda.device(dev):
        out_v = torch.empty((m, k), dtype=v.dtype, device=dev)
        out_i = torch.empty((m, k), dtype=torch.int64, device=dev)
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
        wsb = lib.btk_topk_with_indices_workspace_bytes(m, c, k, dt)
        ws = _ops.workspace(wsb, dev)
        st = lib.btk_topk_with_indices(v.data_ptr(), i.data_ptr(), dt, m, c, k, out_v.data_ptr(),
                                       out_i.data_ptr(), ws.data_ptr(), wsb, flag.data_ptr(),
                                       _ops.stream_handle(dev))
        _ops.raise_status(st, "(topk_with_indices)")
        v_flag = int(flag.item())
        if v_flag & 2 or (check_finite and v_flag & 1):
            _ops.check_flag(flag)
    return TopKResult(values=out_v, indices=out_i)
