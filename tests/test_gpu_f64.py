"""The exact float64 path (the reference's native dtype) against the
reference's own outputs on its own float64 generator, and the committed
reference-side binding (integration/bucketed_topk_b200.py) driving the
UNMODIFIED reference's callers.

Bar: bit-exact indices and float64 value bits (sign of zero included)."""

import hashlib
import os
import sys

import numpy as np
import pytest
import torch

import paper_2412_04358_b200 as btk
from oracle import bucketed_oracle as O
from tests.golden_io import f64_cases, f64_labels

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = f64_cases()


def _asg(s):
    return btk.Assignment.INTERLEAVED if s == "interleaved" else btk.Assignment.CONTIGUOUS


def _same(got_v, got_i, want_v, want_i):
    np.testing.assert_array_equal(np.asarray(got_i), want_i)
    np.testing.assert_array_equal(np.asarray(got_v, np.float64).view(np.int64),
                                  np.asarray(want_v, np.float64).view(np.int64))


@pytest.mark.parametrize("c", CASES, ids=[c["name"] for c in CASES])
def test_f64_reference_inputs(c):
    x = c["gen"]()
    assert hashlib.sha256(x.tobytes()).hexdigest() == c["sha"]
    sch = btk.BucketScheme(c["b"], c["kb"], _asg(c["asg"]))
    r = btk.approx_topk(x, c["k"], sch)           # NumPy float64 in, exact GPU path
    assert r.values.dtype == torch.float64
    _same(r.values.cpu(), r.indices.cpu(), c["values"], c["indices"])
    s1 = btk.stage1(x, sch)
    _same(s1.values.cpu(), s1.indices.cpu(), c["s1_values"], c["s1_indices"])
    e = btk.exact_topk_oracle(x, c["k"])
    _same(e.values.cpu(), e.indices.cpu(), c["ex_values"], c["ex_indices"])


def test_f64_carried_labels():
    L = f64_labels()
    r = btk.topk_with_indices(torch.from_numpy(L["v"]), L["lab"], int(L["k"]))
    _same(r.values.cpu(), r.indices.cpu(), L["values"], L["indices"])


@pytest.mark.parametrize("shape", [(3, 5000, 120, 50, 3), (2, 70000, 9000, 1, 9000), (2, 40000, 700, 40000, 1)])
def test_f64_subnormals_and_signed_zeros(shape):
    m, n, k, b, kb = shape
    rng = np.random.default_rng(n)
    sub = rng.integers(1, 1 << 20, size=(m, n)).astype(np.uint64)   # float64 subnormal bit patterns
    x = sub.view(np.float64) * np.where(rng.random((m, n)) < 0.5, -1.0, 1.0)
    u = rng.random((m, n))
    x[u < 0.2] = 0.0
    x[(u >= 0.2) & (u < 0.4)] = -0.0
    x[(u >= 0.4) & (u < 0.45)] = -1.0
    wv, wi = O.approx_topk(x, k, b, kb)
    r = btk.approx_topk(torch.from_numpy(x).cuda(), k, btk.BucketScheme(b, kb))
    _same(r.values.cpu(), r.indices.cpu(), wv, wi)


def test_f64_nonfinite_raises():
    x = np.zeros((2, 100))
    x[1, 3] = np.nan
    with pytest.raises(btk.NonFiniteInputError):
        btk.approx_topk(x, 10, btk.BucketScheme(10, 1))


def _reference_pkg():
    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "bucketed_topk")):
        pytest.skip("reference package not installed in baseline/_ref")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import bucketed_topk
    return bucketed_topk


def test_integration_binding_drives_reference_callers():
    """install() the binding into the unmodified reference package: its own
    approx_topk / exact / stage1 and its callers (recall.monte_carlo_recall,
    bench.time_selection) now run on the GPU and return identical results."""
    bt = _reference_pkg()
    from integration import bucketed_topk_b200 as b200

    c = CASES[1]
    x = bt.simdata.iid_normal(c["m"], c["n"], seed=c["seed"])
    sch = bt.BucketScheme(b=c["b"], k_b=c["kb"], assignment=bt.Assignment.INTERLEAVED)
    shape = bt.ProblemShape(m=1, n=2048, k=64)
    sch2 = bt.BucketScheme(b=64, k_b=1, assignment=bt.Assignment.INTERLEAVED)
    mc_cpu = bt.monte_carlo_recall(shape, sch2, trials=300, seed=3)
    b200.install(bt)
    try:
        r = bt.approx_topk(x, c["k"], sch)
        assert isinstance(r, bt.TopKResult) and r.values.dtype == np.float64
        _same(r.values, r.indices, c["values"], c["indices"])
        e = bt.exact_topk_oracle(x, c["k"])
        _same(e.values, e.indices, c["ex_values"], c["ex_indices"])
        s1 = bt.approx.stage1(x, sch)
        _same(s1.values, s1.indices, c["s1_values"], c["s1_indices"])
        mc_gpu = bt.recall.monte_carlo_recall(shape, sch2, trials=300, seed=3)
        assert mc_gpu == mc_cpu   # same keyed inputs, bit-identical selections -> identical estimate
        st = bt.bench.time_selection("approx_per_bucket", bt.ProblemShape(m=4, n=4096, k=64), sch2,
                                     warmup=1, iters=3)
        assert st.iterations == 3
        with pytest.raises(bt.ConfigError) as ei:
            bt.approx_topk(x, 100000, sch)
        assert ei.value.code == "k_gt_n"
    finally:
        b200.uninstall(bt)
    assert bt.approx_topk.__module__ == "bucketed_topk.approx"
