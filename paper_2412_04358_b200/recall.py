"""Empirical recall on the GPU (reference recall.py:192-268).

* ``empirical_recall(approx_row, truth_row, k)``  one row, host-side
  (recall.py:203-215; rows are short lists)
* ``empirical_recall_rows(approx, truth)``        per-row recall of two
  (m, k) results; the membership counts run in ``btk_recall_hits``
  (recall.py:218-228)
* ``monte_carlo_recall(shape, scheme, trials, ...)``  mean recall and its
  standard error over trials i.i.d. unit-normal rows (recall.py:231-268):
  the rows come from the reference's keyed Philox generator
  (``simdata.normal_rows``), both selections and the counts run on the GPU
  in float64 (the exact 128-bit-key path), so the per-trial recalls — and
  therefore the mean and standard error — equal the reference's bit for
  bit.  Row generation for the next block overlaps the GPU work of the
  current one.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib, _ops, simdata
from .approx import ExecutionMode, PerBucket, approx_topk
from .core import BucketScheme, ProblemShape, validate
from .exact import ScoredIndex, TopKResult, exact_topk_oracle

__all__ = ["MonteCarloRecall", "empirical_recall", "empirical_recall_rows", "recall_hits",
           "monte_carlo_recall"]


@dataclass(frozen=True)
class MonteCarloRecall:
    """Mean recall over trials with its standard error (recall.py:52-58)."""

    mean_recall: float
    stderr: float
    trials: int


def _indices_of(row) -> np.ndarray:
    if isinstance(row, TopKResult):
        if row.m != 1:
            raise ValueError("pass a single-row result or a row sequence")
        return row.indices[0].cpu().numpy()
    if len(row) and isinstance(row[0], ScoredIndex):
        return np.array([e.index for e in row], dtype=np.int64)
    if isinstance(row, torch.Tensor):
        return row.cpu().numpy().astype(np.int64)
    return np.asarray(row, dtype=np.int64)


def empirical_recall(approx_row, truth_row, k: int) -> float:
    """|approx index set & truth index set| / k for one row."""
    a, t = _indices_of(approx_row), _indices_of(truth_row)
    if a.shape[0] != k or t.shape[0] != k:
        raise ValueError(f"rows must each hold k={k} entries, got {a.shape[0]} and {t.shape[0]}")
    return np.intersect1d(a, t).size / k


def _device_indices(idx, device) -> torch.Tensor:
    t = idx if isinstance(idx, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(idx))
    return t.to(device=device, dtype=torch.int64).contiguous()


def recall_hits(approx_idx, truth_idx) -> torch.Tensor:
    """Device int32 (m,): per row, how many approx indices occur among the
    truth indices.  Asynchronous (no host sync)."""
    dev = approx_idx.device if isinstance(approx_idx, torch.Tensor) and approx_idx.is_cuda else \
        torch.device("cuda", torch.cuda.current_device())
    a = _device_indices(approx_idx, dev)
    t = _device_indices(truth_idx, dev)
    if a.ndim != 2 or tuple(a.shape) != tuple(t.shape):
        raise ValueError("results must have identical (m, k) shapes")
    m, k = a.shape
    with torch.cuda.device(dev):
        hits = torch.empty(m, dtype=torch.int32, device=dev)
        # a size-1 leading dim may carry any stride (e.g. 0 from x[None])
        sa = a.stride(0) if m > 1 else k
        stt = t.stride(0) if m > 1 else k
        st = _lib.load().btk_recall_hits(a.data_ptr(), sa, t.data_ptr(), stt, m, k,
                                         hits.data_ptr(), _ops.stream_handle(dev))
        _ops.raise_status(st, "(recall_hits)")
    return hits


def empirical_recall_rows(approx, truth) -> np.ndarray:
    """Per-row recall of a batch result against the oracle result."""
    if tuple(approx.indices.shape) != tuple(truth.indices.shape):
        raise ValueError("results must have identical (m, k) shapes")
    k = truth.indices.shape[-1]
    return recall_hits(approx.indices, truth.indices).cpu().numpy().astype(np.float64) / k


def monte_carlo_recall(shape: ProblemShape, scheme: BucketScheme, trials: int, seed: int = 0,
                       mode: ExecutionMode = PerBucket(), block_rows: int = 4096, *,
                       device: Optional[torch.device] = None, gen_threads: int = 0) -> MonteCarloRecall:
    """Mean recall over ``trials`` rows (trial t = row t of the seed's
    keyed stream; ``shape.m`` plays no role, as in the reference)."""
    validate(shape, scheme)
    if trials < 1:
        raise ValueError(f"trials must be >= 1, got {trials}")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    n, k = shape.n, shape.k
    blocks = [(d, min(block_rows, trials - d)) for d in range(0, trials, block_rows)]
    threads = gen_threads or min(8, max(1, len(blocks)))

    def gen(b):
        first, rows = b
        return simdata.normal_rows(seed, first, rows, n)

    recalls = np.empty(trials)
    pending = []  # (first, rows, device hits)
    with ThreadPoolExecutor(max_workers=threads) as pool:
        ahead = threads + 1  # blocks generated ahead of the GPU (bounds host memory)
        futures = [pool.submit(gen, b) for b in blocks[:ahead]]
        for i, (first, rows) in enumerate(blocks):
            if i + ahead < len(blocks):
                futures.append(pool.submit(gen, blocks[i + ahead]))
            x = torch.from_numpy(futures[i].result()).to(dev, non_blocking=False)
            futures[i] = None
            got = approx_topk(x, k, scheme, mode)
            want = exact_topk_oracle(x, k)
            pending.append((first, rows, recall_hits(got.indices, want.indices)))
    for first, rows, h in pending:
        recalls[first:first + rows] = h.cpu().numpy().astype(np.float64) / k
    mean = float(recalls.mean())
    stderr = float(recalls.std(ddof=1) / math.sqrt(trials)) if trials > 1 else 0.0
    return MonteCarloRecall(mean_recall=mean, stderr=stderr, trials=trials)
