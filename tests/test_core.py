"""Host-side config layer vs the reference's golden validation codes / rules
(reference tests/test_core.py)."""

import numpy as np
import pytest

from paper_2412_04358_b200.approx import ChunkedMerge, PerBucket, select_mode
from paper_2412_04358_b200.core import (Assignment, BucketScheme, ConfigError, ProblemShape,
                                        bucket_of, bucket_sizes, check_parameters, validate)
from paper_2412_04358_b200.shard import local_rows, row_blocks
from tests.golden_io import load

I, C = Assignment.INTERLEAVED, Assignment.CONTIGUOUS


def test_validation_codes_match_reference():
    z = load("validation.npz")
    for p, code in zip(z["params"], z["codes"]):
        try:
            check_parameters(*(int(v) for v in p))
            got = ""
        except ConfigError as e:
            got = e.code
        assert got == str(code), p


def test_messages_name_constraint():
    with pytest.raises(ConfigError) as e:
        validate(ProblemShape(1, 8, 4), BucketScheme(2, 1, I))
    assert e.value.code == "undersampled" and "b*kb < k" in str(e.value)


def test_bucket_of_examples():
    assert bucket_of(10, 11, 3, I) == 1
    assert bucket_of(10, 11, 3, C) == 2


@pytest.mark.parametrize("asg", [I, C])
def test_sizes_match_fibers(asg):
    rng = np.random.default_rng(7)
    for _ in range(50):
        n = int(rng.integers(1, 200))
        b = int(rng.integers(1, n + 1))
        fib = np.bincount([bucket_of(i, n, b, asg) for i in range(n)], minlength=b)
        assert bucket_sizes(n, b, asg).tolist() == fib.tolist()


def test_select_mode_heuristic():
    assert select_mode(ProblemShape(128, 2**20, 64), BucketScheme(512, 1, I), 1024) == PerBucket()
    assert select_mode(ProblemShape(1, 256, 4), BucketScheme(4, 1, I), 1024) == ChunkedMerge(64)
    assert select_mode(ProblemShape(1, 256, 8), BucketScheme(8, 1, I), 1024) == PerBucket()
    with pytest.raises(ConfigError):
        ChunkedMerge(1)


def test_row_blocks_match_reference_partition():
    # reference exact.py:106-109: linspace partition, empty blocks dropped
    for m in (1, 7, 23, 128, 8192):
        for w in (1, 2, 3, 4, 8, 64):
            blocks = row_blocks(m, w)
            bounds = np.linspace(0, m, max(1, min(w, m)) + 1, dtype=int)
            want = [(a, b) for a, b in zip(bounds[:-1], bounds[1:]) if a < b]
            assert [(s.start, s.stop) for s in blocks] == want
            assert sum(s.stop - s.start for s in blocks) == m
            assert [local_rows(m, w, r) for r in range(len(blocks))] == blocks
