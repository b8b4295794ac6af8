"""GPU parity: the CUDA path (through the C ABI) vs the oracle / golden vectors.

Bar: bit-exact indices and value bits (sign of zero included), every case.
"""

import os

import numpy as np
import pytest
import torch

import paper_2412_04358_b200 as btk
from oracle import bucketed_oracle as O
from tests.golden_io import baseline_cases, load, sha, small_cases

pytestmark = pytest.mark.gpu

I, C = btk.Assignment.INTERLEAVED, btk.Assignment.CONTIGUOUS
DT = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}


def _asg(s):
    return I if s == "interleaved" else C


def _bits(t: torch.Tensor) -> np.ndarray:
    t = t.detach().cpu()
    if t.dtype == torch.float32:
        return t.view(torch.int32).numpy()
    return t.view(torch.int16).numpy()


def _want_bits(v64: np.ndarray, dtype) -> np.ndarray:
    return _bits(torch.from_numpy(np.asarray(v64, np.float64)).to(dtype))


def assert_same(res, want_v, want_i, dtype):
    got_i = res.indices.cpu().numpy()
    assert got_i.dtype == np.int64
    np.testing.assert_array_equal(got_i, want_i)
    np.testing.assert_array_equal(_bits(res.values), _want_bits(want_v, dtype))


def _dtypes_for(x32: np.ndarray):
    out = ["f32"]
    for name, tdt in (("bf16", torch.bfloat16), ("f16", torch.float16)):
        t = torch.from_numpy(x32)
        if torch.equal(t.to(tdt).float(), t) and np.all(np.isfinite(t.to(tdt).float().numpy())):
            out.append(name)
    return out


SMALL = small_cases()


@pytest.mark.parametrize("case", SMALL, ids=[c["name"] for c in SMALL])
def test_small_golden(case):
    x32 = np.ascontiguousarray(case["x"], np.float32)
    for dn in _dtypes_for(x32):
        x = torch.from_numpy(x32).to(DT[dn]).cuda()
        sch = btk.BucketScheme(case["b"], case["kb"], _asg(case["asg"]))
        r = btk.approx_topk(x, case["k"], sch)
        assert_same(r, case["values"], case["indices"], DT[dn])
        s1 = btk.stage1(x, sch)
        np.testing.assert_array_equal(s1.indices.cpu().numpy(), case["s1_indices"])
        np.testing.assert_array_equal(_bits(s1.values), _want_bits(case["s1_values"], DT[dn]))
        np.testing.assert_array_equal(s1.per_bucket, case["s1_per_bucket"])
        e = btk.exact_topk_oracle(x, case["k"])
        assert_same(e, case["ex_values"], case["ex_indices"], DT[dn])


def test_worked_example_literals():
    row = torch.tensor([11.0, 3.0, 10.0, 6.0, 1.0, 4.0, 8.0, 5.0, 2.0, 9.0, 7.0], device="cuda")
    sch = btk.BucketScheme(3, 2, I)
    c = btk.stage1(row, sch)
    assert c.values[0].tolist() == [11, 9, 7, 5, 10, 4]
    assert c.indices[0].tolist() == [0, 9, 10, 7, 2, 5]
    assert c.per_bucket.tolist() == [2, 2, 2]
    r = btk.approx_topk(row, 4, sch)
    assert r.values[0].tolist() == [11, 10, 9, 7] and r.indices[0].tolist() == [0, 2, 9, 10]
    e = btk.exact_topk_oracle(row, 4)
    assert e.values[0].tolist() == [11, 10, 9, 8] and e.indices[0].tolist() == [0, 2, 9, 6]


@pytest.mark.parametrize("case", baseline_cases(), ids=lambda c: c["name"])
def test_baseline_shapes_golden(case):
    x32 = case["gen"]()
    assert sha(x32) == case["sha"]
    dt = torch.float32
    if case["kind"] == "normal_bf16":
        dt = torch.bfloat16
    elif case["kind"] == "normal_f16":
        dt = torch.float16
    x = torch.from_numpy(x32).to(dt).cuda()
    r = btk.approx_topk(x, case["k"], btk.BucketScheme(case["b"], case["kb"], I))
    np.testing.assert_array_equal(r.indices.cpu().numpy(), case["indices"])
    np.testing.assert_array_equal(r.values.float().cpu().numpy(), case["values"])


def test_carried_labels():
    z = load("carried_labels.npz")
    r = btk.topk_with_indices(torch.tensor(z["v"], dtype=torch.float32), z["lab"], int(z["k"]))
    assert r.indices[0].tolist() == [10, 30, 20]
    assert r.values[0].tolist() == [9.0, 9.0, 5.0]
    r = btk.topk_with_indices(torch.tensor(z["v2"]), z["lab2"], int(z["k2"]))
    np.testing.assert_array_equal(r.indices.cpu().numpy(), z["indices2"])
    np.testing.assert_array_equal(r.values.double().cpu().numpy(), z["values2"])


def test_nonfinite_raises():
    for bad in (float("nan"), float("inf"), float("-inf")):
        for dt in DT.values():
            x = torch.zeros(3, 64, dtype=dt, device="cuda")
            x[1, 17] = bad
            with pytest.raises(btk.NonFiniteInputError):
                btk.approx_topk(x, 8, btk.BucketScheme(8, 1, I))
            with pytest.raises(btk.NonFiniteInputError):
                btk.exact_topk_oracle(x, 4)
            # opt-out: no raise
            btk.approx_topk(x, 8, btk.BucketScheme(8, 1, I), check_finite=False)


def test_config_errors_match_reference_codes():
    z = load("validation.npz")
    x = torch.zeros(64, device="cuda")
    for p, code in zip(z["params"], z["codes"]):
        m, n, k, b, kb = (int(v) for v in p)
        got = ""
        try:
            btk.check_parameters(m, n, k, b, kb)
        except btk.ConfigError as e:
            got = e.code
        assert got == str(code)
    with pytest.raises(btk.ConfigError) as e:
        btk.approx_topk(torch.arange(8.0, device="cuda"), 4, btk.BucketScheme(2, 1, I))
    assert e.value.code == "undersampled" and "b*kb < k" in str(e.value)
    del x


def _rand_input(rng, kind, m, n):
    if kind == "normal":
        return rng.standard_normal((m, n), dtype=np.float32)
    if kind == "ties":
        return rng.integers(-3, 4, size=(m, n)).astype(np.float32)
    x = rng.integers(-1, 2, size=(m, n)).astype(np.float32) * 0.0  # +-0 soup
    x[rng.random((m, n)) < 0.2] = 1.0
    return x


@pytest.mark.parametrize("seed", range(6))
def test_random_sweep_vs_oracle(seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(25):
        n = int(rng.integers(1, 5000))
        b = int(rng.integers(1, n + 1))
        cap = -(-n // b)
        kb = int(rng.integers(1, min(cap, 40) + 1))
        k = int(rng.integers(kb, min(n, b * kb) + 1))
        asg = "interleaved" if rng.random() < 0.6 else "contiguous"
        kind = ["normal", "ties", "zeros"][int(rng.integers(3))]
        m = int(rng.integers(1, 5))
        x32 = _rand_input(rng, kind, m, n)
        wv, wi = O.approx_topk(x32, k, b, kb, asg)
        for dn in _dtypes_for(x32):
            x = torch.from_numpy(x32).to(DT[dn]).cuda()
            r = btk.approx_topk(x, k, btk.BucketScheme(b, kb, _asg(asg)))
            assert_same(r, wv, wi, DT[dn])


@pytest.mark.parametrize("n,k,b,kb", [
    (50000, 20000, 1, 20000),      # exact path, long segment, global LSD sort
    (40000, 3000, 1, 3000),        # long segment, select then smem sort
    (70000, 4000, 2, 2000),        # kb > 16 with s > 16384
    (65536, 18000, 9000, 2),       # pool > 16384 -> select_compact + global lsd
    (100003, 5000, 40000, 1),      # ragged, pool > cap, kk fits smem
])
def test_long_segment_paths(n, k, b, kb):
    rng = np.random.default_rng(n + k)
    x32 = rng.standard_normal((2, n), dtype=np.float32)
    x32[:, ::7] = np.round(x32[:, ::7])  # ties
    wv, wi = O.approx_topk(x32, k, b, kb, "interleaved")
    r = btk.approx_topk(torch.from_numpy(x32).cuda(), k, btk.BucketScheme(b, kb, I))
    assert_same(r, wv, wi, torch.float32)


def test_dim_and_strides():
    rng = np.random.default_rng(3)
    x32 = rng.standard_normal((5, 300, 4), dtype=np.float32)
    x = torch.from_numpy(x32).cuda()
    sch = btk.BucketScheme(30, 2, I)
    r = btk.approx_topk(x, 40, sch, dim=1)
    assert tuple(r.values.shape) == (5, 40, 4)
    flat = np.moveaxis(x32, 1, -1).reshape(-1, 300)
    wv, wi = O.approx_topk(flat, 40, 30, 2)
    got_i = r.indices.movedim(1, -1).reshape(-1, 40).cpu().numpy()
    np.testing.assert_array_equal(got_i, wi)
    # a non-contiguous row view
    big = torch.from_numpy(rng.standard_normal((4, 1000), dtype=np.float32)).cuda()
    view = big[:, 100:900]
    wv, wi = O.approx_topk(view.cpu().numpy(), 32, 32, 1)
    r = btk.approx_topk(view, 32, btk.BucketScheme(32, 1, I))
    np.testing.assert_array_equal(r.indices.cpu().numpy(), wi)


def test_full_config1_and_determinism():
    rng = np.random.default_rng(7)
    x32 = rng.standard_normal((128, 65536), dtype=np.float32)
    wv, wi = O.approx_topk(x32, 64, 64, 1, workers=os.cpu_count() or 1)
    x = torch.from_numpy(x32).cuda()
    sch = btk.BucketScheme(64, 1, I)
    r1 = btk.approx_topk(x, 64, sch)
    assert_same(r1, wv, wi, torch.float32)
    op = btk.ApproxTopK(128, 65536, 64, sch, dtype=torch.float32, device="cuda")
    for _ in range(3):
        r = op(x)
        torch.cuda.synchronize()
        assert torch.equal(r.indices, r1.indices) and torch.equal(r.values, r1.values)


def test_full_config4():
    rng = np.random.default_rng(8)
    x32 = rng.standard_normal((4096, 32768), dtype=np.float32)
    xb = torch.from_numpy(x32).to(torch.bfloat16)
    wv, wi = O.approx_topk(xb.float().numpy(), 512, 512, 1, workers=os.cpu_count() or 1)
    r = btk.approx_topk(xb.cuda(), 512, btk.BucketScheme(512, 1, I))
    assert_same(r, wv, wi, torch.bfloat16)


def test_sharded_equals_single():
    rng = np.random.default_rng(9)
    x32 = rng.standard_normal((23, 4096), dtype=np.float32)
    x = torch.from_numpy(x32).cuda()
    sch = btk.BucketScheme(256, 2, I)
    base = btk.approx_topk(x, 256, sch)
    devs = ["cuda:0"] * 3  # same device three times: exercises the partition logic
    r = btk.approx_topk_sharded(x, 256, sch, devices=devs, gather=True)
    assert torch.equal(r.indices, base.indices) and torch.equal(r.values, base.values)
    # default: results stay on the owning devices, one block per device
    parts = btk.approx_topk_sharded(x32, 256, sch, devices=devs)  # host input, copied per block
    assert [p.m for p in parts] == [s.stop - s.start for s in btk.row_blocks(23, 3)]
    assert torch.equal(torch.cat([p.indices for p in parts]), base.indices)
    # N-D input with dim != -1: gathered result has the single-device shape
    x3 = torch.from_numpy(rng.standard_normal((3, 4096, 5), dtype=np.float32)).cuda()
    one = btk.approx_topk(x3, 256, sch, dim=1)
    many = btk.approx_topk(x3, 256, sch, dim=1, devices=devs)
    assert many.values.shape == one.values.shape == (3, 256, 5)
    assert torch.equal(many.indices, one.indices) and torch.equal(many.values, one.values)


_SHAPE_ENVS = [{"BTK_ROWS": "1"}, {"BTK_ROWS": "0", "BTK_S": "1"}, {"BTK_ROWS": "0", "BTK_S": "2"},
               {"BTK_ROWS": "0", "BTK_S": "4"}, {"BTK_ROWS": "0", "BTK_S": "8"},
               {"BTK_ROWS": "0", "BTK_S": "2", "BTK_STAGE_KB": "8", "BTK_NS": "3"}]


@pytest.mark.parametrize("env", _SHAPE_ENVS, ids=lambda e: "-".join(f"{k[4:]}{v}" for k, v in e.items()))
def test_fused_launch_shapes_match_oracle(env, monkeypatch):
    """Every fused kernel / cluster split / ring shape gives the oracle's
    bits (results must not depend on the launch shape: reference
    approx.py:8-16 mode-independence, test_approx.py:194-207)."""
    for k_, v_ in env.items():
        monkeypatch.setenv(k_, v_)
    rng = np.random.default_rng(77)
    cases = [(3, 65536, 64, 64, 1), (2, 32768, 512, 512, 1), (2, 20000, 300, 256, 2),
             (3, 40000, 512, 128, 4), (2, 33000, 256, 64, 8), (4, 8192 + 64, 100, 64, 2),
             (2, 131072, 256, 1024, 1), (3, 4096, 64, 16, 4)]
    for m, n, k, b, kb in cases:
        for kind in ("normal", "ties"):
            x32 = _rand_input(rng, kind, m, n)
            wv, wi = O.approx_topk(x32, k, b, kb)
            for dn in _dtypes_for(x32):
                x = torch.from_numpy(x32).to(DT[dn]).cuda()
                r = btk.approx_topk(x, k, btk.BucketScheme(b, kb, I))
                assert_same(r, wv, wi, DT[dn])


@pytest.mark.parametrize("kind", ["two_values", "one_outlier", "all_equal", "normal_bf16"])
def test_long_segment_skewed_distributions(kind):
    """Exact selection over one 120000-key segment per row (b = 1): the
    long-segment path (radix select + compaction + sort) under adversarially
    skewed value distributions (two values, one outlier, all equal)."""
    rng = np.random.default_rng(5)
    m, n, k = 3, 120000, 60000
    x32 = rng.standard_normal((m, n), dtype=np.float32)
    if kind == "two_values":
        x32[0] = rng.integers(0, 2, size=n).astype(np.float32)
    elif kind == "one_outlier":
        x32[1] = 1.0
        x32[1, 777] = 1e30
    elif kind == "all_equal":
        x32[2] = -2.5
    dt = torch.bfloat16 if kind == "normal_bf16" else torch.float32
    if dt == torch.bfloat16:
        x32 = torch.from_numpy(x32).to(dt).float().numpy()
    wv, wi = O.approx_topk(x32, k, 1, k)  # exact (b = 1): one long segment per row
    r = btk.approx_topk(torch.from_numpy(x32).to(dt).cuda(), k, btk.BucketScheme(1, k, I))
    assert_same(r, wv, wi, dt)
    e = btk.exact_topk_oracle(torch.from_numpy(x32).to(dt).cuda(), k)
    assert_same(e, wv, wi, dt)


@pytest.mark.parametrize("cfg", [(128, 65536, 64, 64, 1, torch.float32), (64, 32768, 512, 512, 1, torch.bfloat16),
                                 (1200, 8192, 256, 256, 1, torch.bfloat16)])
def test_graph_replay_with_pdl_matches_eager(cfg):
    """The bench path: back-to-back launches captured in one CUDA graph
    (programmatic dependent launch edges between them) over rotating
    inputs must give exactly the eager results of the last input."""
    m, n, k, b, kb, dt = cfg
    g = torch.Generator(device="cuda").manual_seed(3)
    bufs = [torch.randn((m, n), generator=g, device="cuda").to(dt) for _ in range(3)]
    sch = btk.BucketScheme(b, kb, I)
    op = btk.ApproxTopK(m, n, k, sch, dtype=dt, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        op.launch(bufs[0])  # warm-up (smem attributes) outside capture
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            for i in range(7):
                op.launch(bufs[i % 3])
        graph.replay()
    torch.cuda.synchronize()
    got_v, got_i = op.values.clone(), op.indices.clone()
    want = btk.approx_topk(bufs[6 % 3], k, sch)
    assert torch.equal(got_i, want.indices) and torch.equal(got_v, want.values)


def _canonical_properties(x, r, k, b, kb):
    """Size-independent checks of one approx_topk result on the device,
    independent of the library's own stage1(): values are the input bits
    at the indices, indices are distinct, rows are in canonical order
    (value desc, index asc on ties), and the selected set is the top-k of
    the per-bucket top-k_b candidates, computed here with plain torch
    (values only, so torch.topk's tie order does not matter):
      * every selected element is >= its bucket's k_b-th largest value and
        no bucket contributes more than k_b elements;
      * the k-th selected value equals the k-th largest candidate value;
      * every candidate strictly above that value is selected.
    Interleaved layout with b | n (reference approx.py:112-131: the buckets
    are the columns of the row viewed as (n/b, b))."""
    m, n = x.shape
    idx, val = r.indices, r.values
    assert idx.shape == (m, k) and idx.dtype == torch.int64
    iv = torch.int16 if x.element_size() == 2 else torch.int32
    assert torch.equal(torch.gather(x, 1, idx).view(iv), val.view(iv))
    s = torch.sort(idx, dim=1).values
    assert bool((s[:, 1:] != s[:, :-1]).all())
    vf = val.float()
    assert bool((vf[:, :-1] >= vf[:, 1:]).all())
    assert bool(((vf[:, :-1] != vf[:, 1:]) | (idx[:, :-1] < idx[:, 1:])).all())
    assert n % b == 0
    for r0 in range(0, m, 256):  # row slabs keep the fp32 temporaries small
        r1 = min(m, r0 + 256)
        xv = x[r0:r1].float().view(r1 - r0, n // b, b)
        top = torch.topk(xv, kb, dim=1).values            # (rows, kb, b) per-bucket top-k_b values
        thr = top[:, kb - 1, :]                            # k_b-th largest per bucket
        cand = top.reshape(r1 - r0, -1)
        kth = torch.topk(cand, k, dim=1).values[:, k - 1]
        sel_v, sel_i = vf[r0:r1], idx[r0:r1]
        bucket = sel_i % b
        assert bool((sel_v >= torch.gather(thr, 1, bucket)).all())
        per_bucket = torch.zeros((r1 - r0, b), dtype=torch.int64, device=x.device)
        per_bucket.scatter_add_(1, bucket, torch.ones_like(bucket))
        assert int(per_bucket.max()) <= kb
        assert torch.equal(sel_v[:, -1], kth)
        assert torch.equal((cand > kth[:, None]).sum(1), (sel_v > kth[:, None]).sum(1))


@pytest.mark.parametrize("name", ["cfg2_kb2", "cfg2_kb4", "cfg2_kb8", "cfg3_r1", "cfg3_r2", "cfg3_r8",
                                  "cfg4", "cfg5"])
def test_full_size_properties_and_row_subset(name):
    """BASELINE sizes (cfg5: 8192 x 2^20 bf16, 17 GB in HBM): canonical
    properties + an independent torch set check on every row, and exact
    oracle parity on a seeded subset of 64 rows (the CPU oracle cannot hold
    cfg5 as float64; rows are independent, reference approx.py:264-282)."""
    from bench import CONFIGS
    dt_s, m, n, k, b, kb, _, _ = CONFIGS[name]
    dt = DT[dt_s]
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.empty((m, n), dtype=dt, device="cuda")
    for r0 in range(0, m, 512):  # generate in slabs (fp32 temporaries stay small)
        r1 = min(m, r0 + 512)
        x[r0:r1] = torch.randn((r1 - r0, n), generator=g, device="cuda").to(dt)
    r = btk.approx_topk(x, k, btk.BucketScheme(b, kb, I))
    torch.cuda.synchronize()
    _canonical_properties(x, r, k, b, kb)
    rows = sorted(torch.randperm(m, generator=torch.Generator().manual_seed(5))[:64].tolist())
    workers = os.cpu_count() or 1
    for c0 in range(0, len(rows), 16):
        sub = rows[c0:c0 + 16]
        x32 = x[sub].float().cpu().numpy()
        wv, wi = O.approx_topk(x32, k, b, kb, workers=workers)
        np.testing.assert_array_equal(r.indices[sub].cpu().numpy(), wi)
        np.testing.assert_array_equal(_bits(r.values[sub]), _want_bits(wv, dt))
    del x, r
    torch.cuda.empty_cache()


def test_cfg5_rows_golden():
    """cfg5 shape at m = 8 rows against the reference's own outputs
    (hash-pinned, tests/golden/cfg5_rows.npz) in bf16 — the s1_vec pool,
    radix select/compaction and global sort path."""
    from tests.golden_io import cfg5_rows, sha_bytes

    c = cfg5_rows()
    x32 = c["gen"]()
    assert sha(x32) == c["sha"]
    x = torch.from_numpy(x32).to(torch.bfloat16).cuda()
    r = btk.approx_topk(x, c["k"], btk.BucketScheme(c["b"], c["kb"], I))
    idx = r.indices.cpu().numpy()
    np.testing.assert_array_equal(idx[0], c["row0_indices"])
    assert sha_bytes(idx.astype(np.int64)) == c["sha_indices"]
    assert sha_bytes(r.values.float().cpu().numpy()) == c["sha_values"]
