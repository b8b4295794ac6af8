"""World-size-2 gloo run of the product's row-sharded logic on CPU.

Each rank owns `local_rows(m, world, rank)` (the reference's `_row_blocks`
partition, exact.py:106-109) and calls the PRODUCT's
`distributed_approx_topk` with the selection stubbed to the CPU oracle
(the kernels need a GPU; the partition, ragged all-gather and
max-over-ranks timing reduction are what is under test), and the gathered
result must equal the single-process result exactly."""

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


def _oracle_select(x, k, scheme, check_finite=True):
    from oracle import bucketed_oracle as O
    from paper_2412_04358_b200 import TopKResult

    v, i = O.approx_topk(x.numpy(), k, scheme.b, scheme.k_b, scheme.assignment.value)
    return TopKResult(values=torch.from_numpy(v.astype(np.float32)), indices=torch.from_numpy(i))


def _worker(rank, world, port, m, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2412_04358_b200 as btk
    from paper_2412_04358_b200.shard import distributed_approx_topk, local_rows, max_over_ranks

    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.standard_normal((m, 512), dtype=np.float32))
    sl = local_rows(m, world, rank)
    scheme = btk.BucketScheme(32, 1, btk.Assignment.INTERLEAVED)
    local = distributed_approx_topk(x[sl], 32, scheme, select=_oracle_select)
    full = distributed_approx_topk(x[sl], 32, scheme, all_gather=True, select=_oracle_select)
    tmax = max_over_ranks(float(rank + 1))
    if rank == 0:
        q.put((tmax, (sl.start, sl.stop), local.indices.shape[0], full.values.numpy(),
               full.indices.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("m,world", [(23, 2), (128, 2), (7, 3)])
def test_row_sharded_matches_single(m, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, q)) for r in range(world)]
    for p in procs:
        p.start()
    tmax, (a, b), local_m, gv, gi = q.get(timeout=180)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert tmax == float(world)
    from oracle import bucketed_oracle as O
    from paper_2412_04358_b200.shard import row_blocks

    assert (a, b) == (row_blocks(m, world)[0].start, row_blocks(m, world)[0].stop)
    assert local_m == b - a
    rng = np.random.default_rng(0)
    x = rng.standard_normal((m, 512), dtype=np.float32)
    wv, wi = O.approx_topk(x, 32, 32, 1)
    np.testing.assert_array_equal(gi, wi)
    np.testing.assert_array_equal(gv, wv.astype(np.float32))
