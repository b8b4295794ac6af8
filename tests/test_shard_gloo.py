"""World-size-2 gloo run of the row-sharded launch logic on CPU.

Each rank owns `local_rows(m, world, rank)` (the reference's `_row_blocks`
partition, exact.py:106-109), selects its rows (here with the oracle —
the GPU kernels need a device; the partition / timing / gather logic is
what is under test), and the bench's max-over-ranks reduction and the
opt-in all-gather must reproduce the single-process result exactly."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import bucketed_oracle as O
    from paper_2412_04358_b200.shard import local_rows

    rng = np.random.default_rng(0)
    x = rng.standard_normal((m, 512), dtype=np.float32)
    sl = local_rows(m, world, rank)
    v, i = O.approx_topk(x[sl], 32, 32, 1)
    # max-over-ranks timing reduction, as in bench.py
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    # opt-in gather of per-rank results (object gather: ragged shards allowed)
    parts = [None] * world
    dist.all_gather_object(parts, (sl.start, sl.stop, i.tolist()))
    if rank == 0:
        q.put((float(t.item()), parts))
    dist.destroy_process_group()


@pytest.mark.parametrize("m", [23, 128])
def test_row_sharded_world2_matches_single(m):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, q)) for r in range(world)]
    for p in procs:
        p.start()
    tmax, parts = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert tmax == 2.0
    from oracle import bucketed_oracle as O

    rng = np.random.default_rng(0)
    x = rng.standard_normal((m, 512), dtype=np.float32)
    _, want = O.approx_topk(x, 32, 32, 1)
    got = np.concatenate([np.array(p[2], dtype=np.int64).reshape(-1, 32) for p in parts])
    assert [(p[0], p[1]) for p in parts] == [(0, m // 2 if m % 2 == 0 else 11), (m // 2 if m % 2 == 0 else 11, m)]
    np.testing.assert_array_equal(got, want)
