"""CPU oracle for the bucketed approximate top-k hot path.

TEST INFRASTRUCTURE ONLY.  This module is a NumPy restatement of the
reference algorithm (`/root/reference/pkg/src/bucketed_topk/`, which is
itself pure NumPy).  It is imported only by `tests/`, by
`__graft_entry__.smoke()` (as the checker) and by `bench.py`'s
`cpu_baseline` / `--impl reference` legs (as the timed CPU arm).  The
product path (`paper_2412_04358_b200`) never imports it and has no CPU
fallback.

Parity pinning: every function below is checked against golden vectors
generated from the real reference (`oracle/make_golden.py` ->
`tests/golden/*.npz`, see `tests/test_oracle_golden.py`) and, when
`/root/reference` is present, against the reference itself on random
inputs.  Status: parity PINNED.

Restated functions (reference file:line):
  as_matrix          exact.py:87-96      float64 upcast, 1-D -> (1, n), finite check
  check_parameters   core.py:84-116      joint validity, codes in order
  bucket_sizes       core.py:134-147
  index_map          approx.py:112-131   (b, s) slot grid, -1 padding
  gather_cube        approx.py:134-139   (m, b, s) cube, -inf padding
  top_slots          approx.py:142-164   k_b<=4: repeated argmax; else stable argsort
  stage1             approx.py:208-242   per-bucket top-k_b + ragged keep mask
  canonical_order    exact.py:130-139    stable by index, then stable by -value
  topk_with_indices  exact.py:142-159
  approx_topk        approx.py:245-282   row blocks over a thread pool
  exact_topk         exact.py:162-173    full stable sort (torch.topk analogue)
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

INTERLEAVED = "interleaved"
CONTIGUOUS = "contiguous"

_SMALL_KB = 4  # approx.py:52


class OracleConfigError(ValueError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class OracleNonFinite(ValueError):
    pass


def as_matrix(scores) -> np.ndarray:
    a = np.asarray(scores, dtype=np.float64)
    if a.ndim == 1:
        a = a[None, :]
    if a.ndim != 2 or a.shape[1] == 0:
        raise ValueError(f"scores must be a non-empty m x n matrix, got {a.shape}")
    if not np.isfinite(a).all():
        raise OracleNonFinite("scores contain NaN or infinity")
    return a


def check_parameters(m, n, k, b, kb) -> None:
    for v in (m, n, k, b, kb):
        if not isinstance(v, (int, np.integer)) or v < 1:
            raise OracleConfigError("nonpositive", "nonpositive")
    if k > n:
        raise OracleConfigError("k_gt_n", "k > n")
    if b > n:
        raise OracleConfigError("b_gt_n", "b > n")
    if kb > min(k, -(-n // b)):
        raise OracleConfigError("kb_range", "kb_range")
    if b * kb < k:
        raise OracleConfigError("undersampled", "b*kb < k")


def bucket_sizes(n: int, b: int, assignment: str) -> np.ndarray:
    if assignment == INTERLEAVED:
        q, r = divmod(n, b)
        s = np.full(b, q, dtype=np.int64)
        s[:r] += 1
        return s
    starts = -(-(np.arange(b + 1, dtype=np.int64) * n) // b)
    return np.diff(starts)


def index_map(n: int, b: int, assignment: str) -> np.ndarray:
    s = -(-n // b)
    sizes = bucket_sizes(n, b, assignment)
    if assignment == INTERLEAVED:
        grid = np.arange(b, dtype=np.int64)[:, None] + b * np.arange(s, dtype=np.int64)[None, :]
        grid[grid >= n] = -1
    else:
        starts = -(-(np.arange(b, dtype=np.int64) * n) // b)
        grid = starts[:, None] + np.arange(s, dtype=np.int64)[None, :]
        grid[np.arange(s)[None, :] >= sizes[:, None]] = -1
    return grid


def gather_cube(a: np.ndarray, grid: np.ndarray) -> np.ndarray:
    cube = a[:, np.maximum(grid, 0)]
    pad = grid < 0
    if pad.any():
        cube[:, pad] = -np.inf
    return cube


def top_slots(cube: np.ndarray, kb: int):
    if kb <= _SMALL_KB:
        work = cube.copy()
        picks = np.empty(cube.shape[:-1] + (kb,), dtype=np.int64)
        vals = np.empty(cube.shape[:-1] + (kb,), dtype=cube.dtype)
        for t in range(kb):
            am = np.argmax(work, axis=-1)[..., None]  # first maximum
            picks[..., t:t + 1] = am
            vals[..., t:t + 1] = np.take_along_axis(work, am, axis=-1)
            np.put_along_axis(work, am, -np.inf, axis=-1)
        return picks, vals
    picks = np.argsort(-cube, axis=-1, kind="stable")[..., :kb].astype(np.int64)
    return picks, np.take_along_axis(cube, picks, axis=-1)


def stage1(a: np.ndarray, b: int, kb: int, assignment: str = INTERLEAVED):
    """(values (m, C) f64, indices (m, C) i64, per_bucket (b,)) in bucket-id order."""
    a = as_matrix(a)
    m, n = a.shape
    grid = index_map(n, b, assignment)
    cube = gather_cube(a, grid)
    picks, vals = top_slots(cube, kb)
    idx = np.take_along_axis(np.broadcast_to(grid[None], cube.shape), picks, axis=2)
    contrib = np.minimum(bucket_sizes(n, b, assignment), kb)
    keep = (np.arange(vals.shape[2])[None, :] < contrib[:, None]).ravel()
    return vals.reshape(m, -1)[:, keep], idx.reshape(m, -1)[:, keep], contrib


def canonical_order(values: np.ndarray, indices: np.ndarray) -> np.ndarray:
    by_index = np.argsort(indices, axis=1, kind="stable")
    v = np.take_along_axis(values, by_index, axis=1)
    by_value = np.argsort(-v, axis=1, kind="stable")
    return np.take_along_axis(by_index, by_value, axis=1)


def topk_with_indices(values, indices, k: int):
    values = np.asarray(values, dtype=np.float64)
    indices = np.asarray(indices, dtype=np.int64)
    if values.ndim == 1:
        values, indices = values[None], indices[None]
    order = canonical_order(values, indices)[:, :k]
    return np.take_along_axis(values, order, axis=1), np.take_along_axis(indices, order, axis=1)


def _row_blocks(m: int, workers: int):
    workers = max(1, min(int(workers), m))
    bounds = np.linspace(0, m, workers + 1, dtype=int)
    return [slice(x, y) for x, y in zip(bounds[:-1], bounds[1:]) if x < y]


def approx_topk(scores, k: int, b: int, kb: int, assignment: str = INTERLEAVED, workers: int = 1):
    """-> (values (m, k) float64, indices (m, k) int64), canonical order."""
    a = as_matrix(scores)
    check_parameters(a.shape[0], a.shape[1], k, b, kb)

    def block(blk):
        v, i, _ = stage1(blk, b, kb, assignment)
        if v.shape[1] < k:
            raise OracleConfigError("insufficient_candidates", "insufficient candidates")
        return topk_with_indices(v, i, k)

    blocks = _row_blocks(a.shape[0], workers)
    if len(blocks) == 1:
        return block(a)
    with ThreadPoolExecutor(max_workers=len(blocks)) as pool:
        parts = list(pool.map(lambda s: block(a[s]), blocks))
    return (np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]))


def exact_topk(scores, k: int, workers: int = 1):
    a = as_matrix(scores)

    def block(blk):
        order = np.argsort(-blk, axis=1, kind="stable")[:, :k].astype(np.int64)
        return np.take_along_axis(blk, order, axis=1), order

    blocks = _row_blocks(a.shape[0], workers)
    parts = [block(a[s]) for s in blocks] if len(blocks) == 1 else list(
        ThreadPoolExecutor(max_workers=len(blocks)).map(lambda s: block(a[s]), blocks))
    return (np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]))


def bytes_moved(m: int, n: int, k: int, value_bytes: int, index_bytes: int = 8) -> int:
    """Paper's minimum traffic (bench.py:154): one read + k (value, index) writes per row."""
    return m * (n * value_bytes + k * (value_bytes + index_bytes))
