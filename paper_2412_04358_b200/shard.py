"""Row-sharded launcher (multi-GPU).

Rows are independent (reference approx.py:264-282), so the reference's
only parallelism — contiguous row blocks over a thread pool
(`_row_blocks`, exact.py:106-109) — maps to contiguous row blocks over
GPUs.  There is no collective on the hot path: every GPU selects its own
rows from its own HBM and keeps the result.  An all-gather of the
(values, indices) is opt-in (``gather=True`` / ``all_gather=True``).

Two entry points:
  * ``approx_topk_sharded``  one process driving several devices (one
    stream each), like the reference's ``workers=`` threads;
  * ``distributed_approx_topk``  one process per GPU under
    ``torch.distributed`` (the bench's launch mode); rank r owns
    ``row_blocks(m, world)[r]``.
"""

from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _ops
from .core import BucketScheme, check_parameters
from .exact import TopKResult

__all__ = ["row_blocks", "approx_topk_sharded", "distributed_approx_topk", "local_rows"]


def row_blocks(m: int, parts: int) -> List[slice]:
    """Contiguous row partition, identical to reference exact.py:106-109."""
    parts = max(1, min(int(parts), m))
    bounds = np.linspace(0, m, parts + 1, dtype=int)
    return [slice(int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:]) if a < b]


def local_rows(m: int, world: int, rank: int) -> slice:
    """Rows rank `rank` owns among `world` shards (empty slice if none)."""
    blocks = row_blocks(m, world)
    return blocks[rank] if rank < len(blocks) else slice(m, m)


def approx_topk_sharded(scores, k: int, scheme: BucketScheme, devices: Sequence, *,
                        dim: int = -1, check_finite: bool = True, gather: bool = True):
    """Split rows over `devices`; each block runs on its own device/stream.

    `scores` is either one tensor / array (rows are copied to their
    owning device) or a list of per-device row blocks already resident.
    Returns one TopKResult on devices[0] when gather=True, else the list of
    per-device TopKResults (no cross-device traffic).
    """
    from .approx import ApproxTopK

    devs = [torch.device(d) for d in devices]
    if isinstance(scores, (list, tuple)):
        parts = list(scores)
        if len(parts) > len(devs):
            raise ValueError("more shards than devices")
    else:
        t = _ops.to_device_tensor(scores, devs[0])
        x, _ = _ops.as_rows(t, dim)
        parts = [x[s] for s in row_blocks(x.shape[0], len(devs))]
    ops, outs = [], []
    for part, dev in zip(parts, devs):
        with torch.cuda.device(dev):
            p = part.to(dev, non_blocking=True) if part.device != dev else part
            p = p if p.stride(-1) == 1 else p.contiguous()
            m, n = p.shape
            check_parameters(m, n, k, scheme.b, scheme.k_b)
            op = ApproxTopK(m, n, k, scheme, dtype=p.dtype, device=dev, row_stride=p.stride(0))
            op.launch(p)
            ops.append(op)
            outs.append(TopKResult(values=op.values, indices=op.indices))
    if check_finite:
        for op in ops:
            with torch.cuda.device(op.device):
                op.check_finite()
    if not gather:
        return outs
    with torch.cuda.device(devs[0]):
        vals = torch.cat([o.values.to(devs[0]) for o in outs])
        idx = torch.cat([o.indices.to(devs[0]) for o in outs])
    return TopKResult(values=vals, indices=idx)


def distributed_approx_topk(local_scores: torch.Tensor, k: int, scheme: BucketScheme, *,
                            all_gather: bool = False, group=None,
                            check_finite: bool = True) -> TopKResult:
    """Per-rank selection of this rank's row block; optional NCCL all-gather.

    Every rank must hold the same number of rows when all_gather=True
    (all_gather_into_tensor needs equal shards).
    """
    import torch.distributed as dist

    from .approx import approx_topk

    res = approx_topk(local_scores, k, scheme, check_finite=check_finite)
    if not all_gather:
        return res
    world = dist.get_world_size(group)
    vals = torch.empty((world * res.values.shape[0], k), dtype=res.values.dtype,
                       device=res.values.device)
    idx = torch.empty((world * res.indices.shape[0], k), dtype=torch.int64,
                      device=res.indices.device)
    dist.all_gather_into_tensor(vals, res.values.contiguous(), group=group)
    dist.all_gather_into_tensor(idx, res.indices.contiguous(), group=group)
    return TopKResult(values=vals, indices=idx)
