"""Row-sharded launcher (multi-GPU).

Rows are independent (reference approx.py:264-282), so the reference's
only parallelism — contiguous row blocks over a thread pool
(`_row_blocks`, exact.py:106-109) — maps to contiguous row blocks over
GPUs.  There is no collective on the hot path: every GPU selects its own
rows from its own HBM and keeps the result.  Gathering the (values,
indices) is opt-in.

Two entry points:
  * ``approx_topk_sharded``  one process driving several devices, like the
    reference's ``workers=`` threads.  Host input is copied block by block
    straight to the owning device (never staged through one GPU); the
    launches are asynchronous, so all devices run concurrently.
  * ``distributed_approx_topk``  one process per GPU under
    ``torch.distributed`` (the bench's launch mode); rank r owns
    ``local_rows(m, world, r)``.  ``all_gather=True`` gathers ragged
    shards (padded to the largest, then trimmed).
"""

from __future__ import annotations

from typing import Callable, List, Optional, Sequence

import numpy as np
import torch

from . import _ops
from .core import BucketScheme, check_parameters
from .exact import TopKResult, _restore

__all__ = ["row_blocks", "local_rows", "approx_topk_sharded", "distributed_approx_topk",
           "gather_rows", "max_over_ranks"]


def row_blocks(m: int, parts: int) -> List[slice]:
    """Contiguous row partition, identical to reference exact.py:106-109."""
    parts = max(1, min(int(parts), m))
    bounds = np.linspace(0, m, parts + 1, dtype=int)
    return [slice(int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:]) if a < b]


def local_rows(m: int, world: int, rank: int) -> slice:
    """Rows rank `rank` owns among `world` shards (empty slice if none)."""
    blocks = row_blocks(m, world)
    return blocks[rank] if rank < len(blocks) else slice(m, m)


def _host_rows(scores, dim):
    """(m, n) row view of a host input plus (lead, orig_ndim) for restore."""
    t = scores if isinstance(scores, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(_ops.host_array(scores)))
    orig_ndim = t.ndim
    x, lead = _ops.as_rows(t, dim)
    return x, lead, orig_ndim


def approx_topk_sharded(scores, k: int, scheme: BucketScheme, devices: Sequence, *,
                        dim: int = -1, check_finite: bool = True, gather: bool = False):
    """Split rows over `devices`; each block runs on its own device.

    `scores` is a host array / CPU tensor (each row block is copied
    directly to its owning device), a CUDA tensor (blocks not already on
    their owner are peer-copied), or a list of per-device row blocks that
    are already resident.  Results stay on their devices: a list of
    per-device TopKResults, unless ``gather=True``, which concatenates
    them on devices[0] and restores the input's leading shape / ``dim``.
    """
    from .approx import _launch

    devs = [torch.device(d) for d in devices]
    lead, orig_ndim = None, 2
    if isinstance(scores, (list, tuple)) and len(scores) and isinstance(scores[0], torch.Tensor):
        parts = list(scores)
        if len(parts) > len(devs):
            raise ValueError("more shards than devices")
        blocks = None
    else:
        if isinstance(scores, torch.Tensor) and scores.is_cuda:
            x = scores
            orig_ndim = x.ndim
            x, lead = _ops.as_rows(x, dim)
        else:
            x, lead, orig_ndim = _host_rows(scores, dim)
        m, n = x.shape
        check_parameters(m, n, k, scheme.b, scheme.k_b)
        blocks = row_blocks(m, len(devs))
        parts = [x[s] for s in blocks]
    launched = []
    for part, dev in zip(parts, devs):
        with torch.cuda.device(dev):
            if part.device != dev:
                # host -> owner (pinned host memory makes this asynchronous)
                part = part.to(dev, non_blocking=part.device.type == "cpu" and part.is_pinned())
            if part.stride(-1) != 1:
                part = part.contiguous()
            m_i, n_i = part.shape
            check_parameters(m_i, n_i, k, scheme.b, scheme.k_b)
            launched.append(_launch(part, k, scheme, check_finite))
    outs = []
    for (vals, idx, flag), dev in zip(launched, devs):
        if flag is not None:
            with torch.cuda.device(dev):
                _ops.check_flag(flag, reset=True)
        outs.append(TopKResult(values=vals, indices=idx))
    if not gather:
        return outs
    with torch.cuda.device(devs[0]):
        vals = torch.cat([o.values.to(devs[0]) for o in outs])
        idx = torch.cat([o.indices.to(devs[0]) for o in outs])
    if lead is not None:
        vals = _restore(vals, lead, dim, orig_ndim)
        idx = _restore(idx, lead, dim, orig_ndim)
    return TopKResult(values=vals, indices=idx)


def gather_rows(t: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather of per-rank (m_r, ...) row blocks in rank order; ragged
    shards (m not divisible by the world size) are padded to the largest
    block for the collective and trimmed after (NCCL over NVLink on GPUs,
    gloo on CPU)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    cnt = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt, group=group)
    sizes = [int(c.item()) for c in cnts]
    mx = max(sizes)
    pad = t
    if t.shape[0] < mx:
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad.contiguous(), group=group)
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)])


def max_over_ranks(v: float, group=None, device=None) -> float:
    """The bench's step time: the max over ranks (float64 all-reduce)."""
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return v
    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def distributed_approx_topk(local_scores, k: int, scheme: BucketScheme, *,
                            all_gather: bool = False, group=None, check_finite: bool = True,
                            select: Optional[Callable] = None) -> TopKResult:
    """Per-rank selection of this rank's row block; optional all-gather.

    ``select(local_scores, k, scheme, check_finite=...) -> TopKResult``
    defaults to :func:`approx_topk` on this rank's GPU (it is injectable so
    the gather logic runs under gloo on CPU in the tests).  Without
    ``all_gather`` the result stays on the rank's device.
    """
    if select is None:
        from .approx import approx_topk as select
    res = select(local_scores, k, scheme, check_finite=check_finite)
    if not all_gather:
        return res
    return TopKResult(values=gather_rows(res.values, group), indices=gather_rows(res.indices, group))
