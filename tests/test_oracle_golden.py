"""Pin the NumPy oracle against golden vectors produced by the real reference.

CPU-only.  If the oracle disagrees with the reference's own outputs, every
GPU parity claim built on it is void, so this runs first.
"""

import os

import numpy as np
import pytest

from oracle import bucketed_oracle as O
from tests.golden_io import baseline_cases, load, sha, small_cases

SMALL = small_cases()


@pytest.mark.parametrize("case", SMALL, ids=[c["name"] for c in SMALL])
def test_oracle_small_cases(case):
    x = case["x"]
    v, i = O.approx_topk(x, case["k"], case["b"], case["kb"], case["asg"])
    assert np.array_equal(i, case["indices"])
    assert np.array_equal(v.view(np.int64), case["values"].view(np.int64))  # sign of zero too
    sv, si, pb = O.stage1(x, case["b"], case["kb"], case["asg"])
    assert np.array_equal(si, case["s1_indices"])
    assert np.array_equal(sv.view(np.int64), case["s1_values"].view(np.int64))
    assert np.array_equal(pb, case["s1_per_bucket"])
    ev, ei = O.exact_topk(x, case["k"])
    assert np.array_equal(ei, case["ex_indices"])
    assert np.array_equal(ev.view(np.int64), case["ex_values"].view(np.int64))


def test_worked_example_literals():
    # reference tests: test_approx.py:31-35, 101-105; test_exact.py:20-23; test_cli.py:41
    row = [11.0, 3.0, 10.0, 6.0, 1.0, 4.0, 8.0, 5.0, 2.0, 9.0, 7.0]
    v, i, pb = O.stage1(row, 3, 2)
    assert v[0].tolist() == [11, 9, 7, 5, 10, 4]
    assert i[0].tolist() == [0, 9, 10, 7, 2, 5]
    assert pb.tolist() == [2, 2, 2]
    v, i = O.approx_topk(row, 4, 3, 2)
    assert v[0].tolist() == [11, 10, 9, 7] and i[0].tolist() == [0, 2, 9, 10]
    v, i = O.exact_topk(row, 4)
    assert v[0].tolist() == [11, 10, 9, 8] and i[0].tolist() == [0, 2, 9, 6]


def test_oracle_carried_labels():
    z = load("carried_labels.npz")
    v, i = O.topk_with_indices(z["v"], z["lab"], int(z["k"]))
    assert v.tolist() == z["values"].tolist() and i.tolist() == z["indices"].tolist()
    assert i[0].tolist() == [10, 30, 20]
    v, i = O.topk_with_indices(z["v2"], z["lab2"], int(z["k2"]))
    assert np.array_equal(i, z["indices2"]) and np.array_equal(v, z["values2"])


def test_oracle_validation_codes():
    z = load("validation.npz")
    for p, code in zip(z["params"], z["codes"]):
        try:
            O.check_parameters(*(int(t) for t in p))
            got = ""
        except O.OracleConfigError as e:
            got = e.code
        assert got == str(code), (p, code, got)


@pytest.mark.parametrize("case", baseline_cases(), ids=lambda c: c["name"])
def test_oracle_baseline_shapes(case):
    x = case["gen"]()
    assert sha(x) == case["sha"], "input generator drifted; regenerate fixtures"
    v, i = O.approx_topk(x, case["k"], case["b"], case["kb"], workers=os.cpu_count() or 1)
    assert np.array_equal(i, case["indices"])
    assert np.array_equal(v.astype(np.float32), case["values"])


def test_bytes_moved_known_answer():
    # reference test_bench.py:81-88
    assert O.bytes_moved(128, 2**20, 64, 4, 8) == 536_969_216


def test_oracle_cfg5_rows_golden():
    """cfg5 (b = 65536, k_b = 2, k = 65536 of 2^20) at m = 8, hashed outputs."""
    from tests.golden_io import cfg5_rows, sha_bytes

    c = cfg5_rows()
    x = c["gen"]()
    assert sha(x) == c["sha"]
    v, i = O.approx_topk(x, c["k"], c["b"], c["kb"], workers=os.cpu_count() or 1)
    np.testing.assert_array_equal(i[0], c["row0_indices"])
    assert sha_bytes(i.astype(np.int64)) == c["sha_indices"]
    assert sha_bytes(v.astype(np.float32)) == c["sha_values"]


def test_oracle_f64_iid_golden():
    """The oracle on the reference's own float64 inputs (keyed Philox,
    simdata.py:38-66) against the reference's outputs."""
    import hashlib

    from tests.golden_io import f64_cases, f64_labels

    for c in f64_cases():
        x = c["gen"]()
        assert hashlib.sha256(x.tobytes()).hexdigest() == c["sha"], c["name"]
        v, i = O.approx_topk(x, c["k"], c["b"], c["kb"], c["asg"])
        assert np.array_equal(i, c["indices"]) and np.array_equal(v.view(np.int64), c["values"].view(np.int64))
        sv, si, _ = O.stage1(x, c["b"], c["kb"], c["asg"])
        assert np.array_equal(si, c["s1_indices"]) and np.array_equal(sv, c["s1_values"])
        ev, ei = O.exact_topk(x, c["k"])
        assert np.array_equal(ei, c["ex_indices"]) and np.array_equal(ev, c["ex_values"])
    L = f64_labels()
    v, i = O.topk_with_indices(L["v"], L["lab"], int(L["k"]))
    assert np.array_equal(i, L["indices"]) and np.array_equal(v.view(np.int64), L["values"].view(np.int64))
