"""Two-stage bucketed approximate top-k on the B200 (the hot path).

Drop-in mirror of reference `approx.py` (same names, argument order, error
classes and codes):

* ``approx_topk(scores, k, scheme, mode=PerBucket(), workers=1)`` -> approx.py:245-282
* ``stage1(scores, scheme, mode=PerBucket())``                      -> approx.py:208-242
* ``Stage1Candidates`` / ``PerBucket`` / ``ChunkedMerge``            -> approx.py:58-109
* ``select_mode(shape, scheme, lanes)``                              -> approx.py:285-297

Additions: ``dim`` (the reference always reduces the last axis),
``check_finite`` (the NaN/inf check costs one device->host sync), and
``devices`` (row-sharding over GPUs, the analogue of ``workers``).
``mode`` and ``workers`` are validated and accepted; the output never
depends on them (reference approx.py:8-16 contract).

``ApproxTopK`` is the prepared form (fixed shape, preallocated outputs and
workspace, no host sync): one C-ABI call per invocation, CUDA-graph safe.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Union

import numpy as np
import torch

from . import _lib, _ops
from .core import (Assignment, BucketScheme, ConfigError, ProblemShape, bucket_sizes,
                   check_parameters, max_bucket_size)
from .exact import ScoredIndex, TopKResult, _restore

__all__ = ["PerBucket", "ChunkedMerge", "ExecutionMode", "Stage1Candidates", "stage1",
           "approx_topk", "select_mode", "ApproxTopK"]

_CHUNK_THRESHOLD = 64  # reference approx.py:55


@dataclass(frozen=True)
class PerBucket:
    """One logical worker per (row, bucket)."""


@dataclass(frozen=True)
class ChunkedMerge:
    """Buckets split into interleaved chunks, merged once per bucket."""

    chunks_per_bucket: int

    def __post_init__(self):
        c = self.chunks_per_bucket
        if not isinstance(c, (int, np.integer)) or c < 2:
            raise ConfigError("chunks_range", f"chunks_per_bucket must be >= 2, got {c!r}")


ExecutionMode = Union[PerBucket, ChunkedMerge]


@dataclass(frozen=True)
class Stage1Candidates:
    """Per-row Stage-1 survivors in bucket-id order (reference approx.py:83-109)."""

    values: torch.Tensor
    indices: torch.Tensor
    per_bucket: np.ndarray

    @property
    def m(self) -> int:
        return self.values.shape[0]

    @property
    def count_per_row(self) -> int:
        return self.values.shape[1]

    def row(self, r: int) -> List[ScoredIndex]:
        return [ScoredIndex(float(v), int(i))
                for v, i in zip(self.values[r].float().tolist(), self.indices[r].tolist())]


def _layout(assignment: Assignment) -> int:
    if assignment is Assignment.INTERLEAVED:
        return _lib.BTK_INTERLEAVED
    if assignment is Assignment.CONTIGUOUS:
        return _lib.BTK_CONTIGUOUS
    raise ConfigError("assignment", f"unknown assignment {assignment!r}")


def _check_mode(mode) -> None:
    if not isinstance(mode, (PerBucket, ChunkedMerge)):
        raise TypeError(f"mode must be PerBucket() or ChunkedMerge(c), got {mode!r}")


class ApproxTopK:
    """Prepared bucketed top-k for a fixed (m, n, dtype, device) batch.

    Allocates outputs and workspace once; ``__call__(x)`` is a single
    asynchronous C-ABI launch on the current stream (no host sync), so it
    can be timed back to back or captured in a CUDA graph.
    """

    def __init__(self, m: int, n: int, k: int, scheme: BucketScheme, dtype=torch.float32,
                 device="cuda", row_stride: Optional[int] = None, inputs_ready: bool = False):
        check_parameters(m, n, k, scheme.b, scheme.k_b)
        self.m, self.n, self.k, self.scheme = m, n, k, scheme
        self.device = torch.device(device)
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.dtype = dtype
        self.row_stride = n if row_stride is None else row_stride
        self.lib = _lib.load()
        self.dt = _ops.dtype_code(torch.empty(0, dtype=dtype))
        self.layout = _layout(scheme.assignment)
        # BTK_INPUT_READY (include/btk.h): the caller promises that inputs are
        # never written by the work queued just before a launch (independent
        # batches resident in HBM), so back-to-back launches may overlap: each
        # streams its input while the previous one drains and waits for it
        # only before writing.  Results are identical either way.
        self.launch_flags = _lib.BTK_INPUT_READY if inputs_ready else 0
        with torch.cuda.device(self.device):
            self.values = torch.empty((m, k), dtype=dtype, device=self.device)
            self.indices = torch.empty((m, k), dtype=torch.int64, device=self.device)
            self.flag = torch.zeros(1, dtype=torch.int32, device=self.device)
            # workspace of the plan that will run for 16-byte aligned inputs
            # of this stride (the fused kernels need none); a misaligned
            # input is rejected at launch rather than silently re-planned
            self.ws_bytes = self.lib.btk_plan_workspace_bytes(
                256, self.row_stride, self.dt, m, n, k, scheme.b, scheme.k_b, self.layout)
            self.ws = _ops.workspace(self.ws_bytes, self.device)

    @property
    def fused(self) -> bool:
        return bool(self.lib.btk_uses_fused_path(self.m, self.n, self.k, self.scheme.b,
                                                 self.scheme.k_b, self.dt, self.layout,
                                                 self.row_stride))

    def launch(self, x: torch.Tensor, stream: Optional[int] = None) -> None:
        if x.dtype != self.dtype or x.device != self.device or x.stride(-1) != 1:
            raise ValueError("input does not match the prepared dtype/device/layout")
        if tuple(x.shape) != (self.m, self.n) or (self.m > 1 and x.stride(0) != self.row_stride):
            raise ValueError(f"input shape/stride {tuple(x.shape)}/{x.stride()} does not match "
                             f"prepared ({self.m}, {self.n}) stride {self.row_stride}")
        if x.data_ptr() % 16:
            raise ValueError("prepared ApproxTopK needs a 16-byte aligned input (use approx_topk "
                             "for arbitrary views)")
        with torch.cuda.device(self.device):  # launches (and the exchange's side stream) on the op's GPU
            st = self.lib.btk_approx_topk_flags(
                x.data_ptr(), self.row_stride, self.dt, self.m, self.n, self.k, self.scheme.b,
                self.scheme.k_b, self.layout, self.values.data_ptr(), self.indices.data_ptr(),
                self.ws.data_ptr(), self.ws_bytes, self.flag.data_ptr(), self.launch_flags,
                _ops.stream_handle(self.device) if stream is None else stream)
        _ops.raise_status(st, "(approx_topk)")

    def __call__(self, x: torch.Tensor) -> TopKResult:
        self.launch(x)
        return TopKResult(values=self.values, indices=self.indices)

    def check_finite(self) -> None:
        """Raise NonFiniteInputError if any launch since the last check saw
        NaN/inf (one device->host sync).  The flag is cleared on read, so
        each check covers the launches after the previous one."""
        _ops.check_flag(self.flag, reset=True)


def approx_topk(scores, k: int, scheme: BucketScheme, mode: ExecutionMode = PerBucket(),
                workers: int = 1, *, dim: int = -1, check_finite: bool = True,
                devices: Optional[Sequence] = None) -> TopKResult:
    """Bucketed approximate top-k (GPU).  See module docstring.

    One kernel launch on the fused path (plus, when ``check_finite``, one
    4-byte device->host read of the non-finite flag); outputs are fresh
    tensors from the caching allocator, the workspace (generic path only)
    too."""
    _check_mode(mode)
    if devices is not None and len(devices) > 1:
        from .shard import approx_topk_sharded
        return approx_topk_sharded(scores, k, scheme, devices=devices, dim=dim,
                                   check_finite=check_finite, gather=True)
    del workers
    dev0 = devices[0] if devices else None
    t = _ops.to_device_tensor(scores, dev0)
    orig_ndim = t.ndim
    x, lead = _ops.as_rows(t, dim)
    m, n = x.shape
    check_parameters(m, n, k, scheme.b, scheme.k_b)
    vals, idx, flag = _launch(x, k, scheme, check_finite)
    if flag is not None:
        with torch.cuda.device(x.device):
            _ops.check_flag(flag, reset=True)
    return TopKResult(values=_restore(vals, lead, dim, orig_ndim),
                      indices=_restore(idx, lead, dim, orig_ndim))


def _launch(x: torch.Tensor, k: int, scheme: BucketScheme, check_finite: bool):
    """Asynchronous launch on x's device / current stream: fresh (m, k)
    outputs, no host sync.  Returns (values, indices, flag or None)."""
    m, n = x.shape
    lib = _lib.load()
    dt = _ops.dtype_code(x)
    lay = _layout(scheme.assignment)
    dev = x.device
    with torch.cuda.device(dev):
        vals = torch.empty((m, k), dtype=x.dtype, device=dev)
        idx = torch.empty((m, k), dtype=torch.int64, device=dev)
        wsb = lib.btk_plan_workspace_bytes(x.data_ptr(), x.stride(0), dt, m, n, k, scheme.b,
                                           scheme.k_b, lay)
        ws = _ops.workspace(wsb, dev) if wsb else None
        flag = _ops.device_flag(dev) if check_finite else None
        st = lib.btk_approx_topk(x.data_ptr(), x.stride(0), dt, m, n, k, scheme.b, scheme.k_b,
                                 lay, vals.data_ptr(), idx.data_ptr(),
                                 ws.data_ptr() if ws is not None else None, wsb,
                                 flag.data_ptr() if flag is not None else None,
                                 _ops.stream_handle(dev))
        _ops.raise_status(st, "(approx_topk)")
    return vals, idx, flag


def stage1(scores, scheme: BucketScheme, mode: ExecutionMode = PerBucket(), *,
           check_finite: bool = True) -> Stage1Candidates:
    """Per-bucket top-k_b, candidates in bucket-id order (reference approx.py:208-242)."""
    _check_mode(mode)
    t = _ops.to_device_tensor(scores)
    x, _ = _ops.as_rows(t, -1)
    m, n = x.shape
    b, kb = scheme.b, scheme.k_b
    if not isinstance(b, (int, np.integer)) or not (1 <= b <= n):
        raise ConfigError("b_gt_n", f"b must be in 1..n (b={b}, n={n})")
    cap = max_bucket_size(n, b)
    if not isinstance(kb, (int, np.integer)) or not (1 <= kb <= cap):
        raise ConfigError("kb_range", f"k_b out of range (k_b={kb}, allowed 1..ceil(n/b)={cap})")
    lib = _lib.load()
    dt = _ops.dtype_code(x)
    lay = _layout(scheme.assignment)
    C = int(lib.btk_stage1_count(n, b, kb, lay))
    dev = x.device
    with torch.cuda.device(dev):
        vals = torch.empty((m, C), dtype=x.dtype, device=dev)
        idx = torch.empty((m, C), dtype=torch.int64, device=dev)
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
        wsb = lib.btk_stage1_workspace_bytes(m, n, b, kb, dt, lay)
        ws = _ops.workspace(wsb, dev)
        st = lib.btk_stage1(x.data_ptr(), x.stride(0), dt, m, n, b, kb, lay, vals.data_ptr(),
                            idx.data_ptr(), ws.data_ptr(), wsb, flag.data_ptr(),
                            _ops.stream_handle(dev))
        _ops.raise_status(st, "(stage1)")
        if check_finite:
            _ops.check_flag(flag)
    per_bucket = np.minimum(bucket_sizes(n, b, scheme.assignment), kb)
    return Stage1Candidates(values=vals, indices=idx, per_bucket=per_bucket)


def select_mode(shape: ProblemShape, scheme: BucketScheme, lanes: int) -> ExecutionMode:
    """Reference heuristic (approx.py:285-297); on the GPU the launch shape
    is chosen internally and the result is mode-independent."""
    if shape.m * scheme.b >= lanes:
        return PerBucket()
    if max_bucket_size(shape.n, scheme.b) < _CHUNK_THRESHOLD:
        return PerBucket()
    return ChunkedMerge(_CHUNK_THRESHOLD)
