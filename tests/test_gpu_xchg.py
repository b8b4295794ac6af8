"""The exchange family (btk_xchg.cu, BTK_FAM_XCHG) against the oracle, both
pipelines: the batched cluster-free one (16-bit default: xb_split /
xb_part / xb_sort) and the 16-CTA cluster kernel (BTK_XB=0).  Every 16-bit
dtype and k_b served, thresholds inside and at the pool edge, tie-heavy
rows that take the fallback kernel next to rows that do not, subnormals /
signed zeros, several batches (double-buffered, partition and sort on two
streams, inside a CUDA graph), and the fp32 64-bit-key cluster variant
forced with BTK_XC=1.

Reference: approx.py:208-282 (stage1 + topk_with_indices),
exact.py:130-159 (canonical order).
"""

import os

import numpy as np
import pytest
import torch

import paper_2412_04358_b200 as btk
from paper_2412_04358_b200 import _lib
from oracle import bucketed_oracle as O
from tests.special_inputs import TORCH, special, to_dtype

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["batched", "cluster"])
def pipe(request, monkeypatch):
    if request.param == "cluster":
        monkeypatch.setenv("BTK_XB", "0")
    else:
        monkeypatch.delenv("BTK_XB", raising=False)
    return request.param

_DTC = {"f32": _lib.BTK_F32, "bf16": _lib.BTK_BF16, "f16": _lib.BTK_F16}


def _bits(t):
    t = t.detach().cpu()
    return t.view(torch.int32 if t.dtype == torch.float32 else torch.int16).numpy()


def _family(m, n, k, b, kb, dn):
    return _lib.load().btk_kernel_family(m, n, k, b, kb, _DTC[dn], _lib.BTK_INTERLEAVED, n)


def _check(x32, dn, k, b, kb):
    x = to_dtype(x32, dn).cuda()
    r = btk.approx_topk(x, k, btk.BucketScheme(b, kb))
    wv, wi = O.approx_topk(x32, k, b, kb)
    np.testing.assert_array_equal(r.indices.cpu().numpy(), wi)
    want = _bits(torch.from_numpy(np.asarray(wv, np.float64)).to(TORCH[dn]))
    np.testing.assert_array_equal(_bits(r.values), want)


def _fallback_rows(x, k, b, kb):
    """Rows the exchange handed to its fallback kernel (the device-side
    list at the head of a prepared op's workspace: count, then row ids)."""
    m, n = x.shape
    op = btk.ApproxTopK(m, n, k, btk.BucketScheme(b, kb), dtype=x.dtype, device=x.device)
    op.launch(x)
    torch.cuda.synchronize()
    cnt = int(op.ws[:4].view(torch.int32).item())
    rows = sorted(op.ws[256:256 + 4 * m].view(torch.int32)[:cnt].cpu().tolist())
    return rows, op


# (m, n, k, b, kb): cfg5 rows, thresholds at 1/2, ~0.6, the whole pool, k_b 1/2/4
SHAPES = [
    (3, 1 << 20, 65536, 65536, 2),
    (2, 262144, 20000, 16384, 2),
    (3, 131072, 12000, 16384, 2),
    (2, 262144, 32768, 16384, 2),   # k = the whole pool (select all)
    (2, 262144, 9000, 32768, 1),
    (2, 262144, 30000, 8192, 4),
    (5, 524288, 30000, 32768, 1),
]


@pytest.mark.parametrize("dn", ["bf16", "f16"])
def test_xchg_normal_and_ties(dn, pipe):
    rng = np.random.default_rng(11)
    for (m, n, k, b, kb) in SHAPES:
        assert _family(m, n, k, b, kb, dn) == _lib.BTK_FAM_XCHG, (m, n, k, b, kb)
        x32 = torch.from_numpy(rng.standard_normal((m, n), dtype=np.float32)).to(TORCH[dn]).float().numpy()
        _check(x32, dn, k, b, kb)
        ties = np.round(x32 * 4) / 4  # few distinct values: large equal-value groups
        _check(ties, dn, k, b, kb)


@pytest.mark.parametrize("dn", ["bf16", "f16"])
def test_xchg_special_values(dn, pipe):
    rng = np.random.default_rng(12)
    for (m, n, k, b, kb) in SHAPES[:4]:
        for kind in ("subnormal", "subnormal_ties", "pm0"):
            _check(special(rng, kind, m, n, dn), dn, k, b, kb)


@pytest.mark.parametrize("dn", ["bf16", "f16"])
def test_xchg_fallback_rows_mixed(dn, pipe):
    """Tie-heavy rows overflow an owner and go to the fallback kernel;
    normal rows in the same batch stay in-cluster; both are exact."""
    rng = np.random.default_rng(13)
    m, n, k, b, kb = 4, 262144, 20000, 16384, 2
    x32 = torch.from_numpy(rng.standard_normal((m, n), dtype=np.float32)).to(TORCH[dn]).float().numpy()
    x32[1] = 0.5          # one value everywhere: every key in one owner
    x32[3, ::2] = -0.0    # half signed zeros, half normals
    _check(x32, dn, k, b, kb)
    rows, _ = _fallback_rows(to_dtype(x32, dn).cuda(), k, b, kb)
    assert 0 not in rows and 2 not in rows and 1 in rows, rows


def test_xchg_cfg5_rows_stay_in_cluster(pipe):
    """N(0,1) cfg5 rows: no fallback (the splitter margins hold)."""
    torch.manual_seed(5)
    x = torch.randn(200 if pipe == "batched" else 32, 1 << 20, device="cuda").to(torch.bfloat16)
    rows, op = _fallback_rows(x, 65536, 65536, 2)
    assert rows == [], rows
    # and the outputs equal the chunked-pool path's on the same input
    import os
    os.environ["BTK_XC"] = "0"
    try:
        ref = btk.approx_topk(x, 65536, btk.BucketScheme(65536, 2))
    finally:
        del os.environ["BTK_XC"]
    assert torch.equal(op.indices, ref.indices)
    assert torch.equal(op.values.view(torch.int16), ref.values.view(torch.int16))


@pytest.mark.parametrize("streams", ["1", "0"])
def test_xb_several_batches(monkeypatch, streams):
    """Batches of 2 rows (BTK_XB_ROWS=2): double-buffered partition / sort
    buffers, the sorts on the side stream (or all on one stream), a
    tie-heavy fallback row in the middle batch."""
    monkeypatch.setenv("BTK_XB_ROWS", "2")
    monkeypatch.setenv("BTK_XB_STREAMS", streams)
    rng = np.random.default_rng(15)
    for dn in ("bf16", "f16"):
        m, n, k, b, kb = 7, 262144, 20000, 16384, 2
        x32 = torch.from_numpy(rng.standard_normal((m, n), dtype=np.float32)).to(TORCH[dn]).float().numpy()
        x32[3] = 0.25
        _check(x32, dn, k, b, kb)
        rows, _ = _fallback_rows(to_dtype(x32, dn).cuda(), k, b, kb)
        assert rows == [3], rows


def test_xchg_fp32_forced(monkeypatch):
    """fp32 through the 64-bit-key variant (BTK_XC=1; not the default)."""
    monkeypatch.setenv("BTK_XC", "1")
    rng = np.random.default_rng(14)
    for (m, n, k, b, kb) in [(3, 65536, 16384, 8192, 2), (2, 65536, 16384, 2048, 8), (3, 65536, 10000, 8192, 2)]:
        assert _family(m, n, k, b, kb, "f32") == _lib.BTK_FAM_XCHG
        x32 = rng.standard_normal((m, n), dtype=np.float32)
        _check(x32, "f32", k, b, kb)
        _check(special(rng, "pm0", m, n, "f32"), "f32", k, b, kb)


@pytest.mark.parametrize("shape", [
    (3, 65536, 64, 64, 1, torch.float32, None),          # fused_narrow (cluster, TMA ring)
    (128, 65536, 64, 64, 1, torch.float32, None),        # fused_narrow, one CTA per row when ready (cfg1)
    (128, 1 << 20, 256, 512, 2, torch.bfloat16, None),   # fused_narrow, deep rows (cfg3), 32 KB stages when ready
    (1200, 2048, 64, 64, 1, torch.bfloat16, None),       # fused_rows (one warp per row)
    (2, 65536, 16384, 8192, 2, torch.float32, None),     # fused_wide
    (2, 262144, 20000, 16384, 2, torch.bfloat16, "0"),   # fused_xchg (cluster)
    (2, 262144, 20000, 16384, 2, torch.bfloat16, None),  # batched exchange, one batch
    (5, 262144, 20000, 16384, 2, torch.bfloat16, "2"),   # batched exchange, 3 batches, 2 streams
], ids=["narrow", "narrow-solo", "narrow-deep", "rows", "wide", "xchg", "xb", "xb-batches"])
def test_inputs_ready_overlapped_launches_equal_serial(shape, monkeypatch):
    """BTK_INPUT_READY launches back to back (eager and in a CUDA graph)
    over rotating buffers: every step's outputs equal the conservative
    launch's, and the last write wins (writes still wait for the
    predecessor)."""
    m, n, k, b, kb, dt, xb = shape
    if xb == "0":
        monkeypatch.setenv("BTK_XB", "0")
    elif xb is not None:
        monkeypatch.setenv("BTK_XB_ROWS", xb)
    xs = [torch.randn(m, n, device="cuda").to(dt) for _ in range(3)]
    sch = btk.BucketScheme(b, kb)
    ready = btk.ApproxTopK(m, n, k, sch, dtype=dt, device="cuda", inputs_ready=True)
    dep = btk.ApproxTopK(m, n, k, sch, dtype=dt, device="cuda")
    want = []
    for x in xs:
        dep.launch(x)
        want.append((dep.values.clone(), dep.indices.clone()))
    got = []
    for i in range(7):
        ready.launch(xs[i % 3])
        got.append((ready.values.clone(), ready.indices.clone()))
    torch.cuda.synchronize()
    for i, (v, ix) in enumerate(got):
        assert torch.equal(ix, want[i % 3][1]) and torch.equal(v, want[i % 3][0]), i
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ready.launch(xs[0])
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(5):
                ready.launch(xs[i % 3])
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(ready.indices, want[4 % 3][1]) and torch.equal(ready.values, want[4 % 3][0])


def _xchg_shapes(seed, count):
    """Seeded shapes the exchange family serves: s below / above 16 and not a
    multiple of the load batch, thresholds from a handful of keys to the
    whole pool, k_b 1/2/4, batches that do not divide m."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        b = int(rng.choice([4096, 8192, 16384, 32768, 65536]))
        kb = int(rng.choice([1, 2, 4]))
        s = int(rng.choice([1, 2, 3, 5, 7, 8, 9, 13, 16, 17, 24, 31]))
        P = b * kb
        if P <= 16384 or s < kb or b // 16 * kb > 8192:
            continue
        k = int(min(P, 16 * 4096, max(1, rng.integers(1, P + 1) if rng.random() < 0.7 else P)))
        m = int(rng.integers(1, 6))
        out.append((m, s * b, k, b, kb))
    return out


@pytest.mark.parametrize("dn", ["bf16", "f16"])
def test_xb_random_shapes(dn, monkeypatch):
    """Randomised exchange-family shapes through the batched pipeline
    (several batch sizes) against the oracle, normal and tie-heavy rows."""
    rng = np.random.default_rng(21 if dn == "bf16" else 22)
    for i, (m, n, k, b, kb) in enumerate(_xchg_shapes(31 if dn == "bf16" else 32, 10)):
        assert _family(m, n, k, b, kb, dn) == _lib.BTK_FAM_XCHG, (m, n, k, b, kb)
        monkeypatch.setenv("BTK_XB_ROWS", str(1 + i % 3))
        x32 = torch.from_numpy(rng.standard_normal((m, n), dtype=np.float32)).to(TORCH[dn]).float().numpy()
        if i % 2:
            x32 = np.round(x32 * 8) / 8
        if i % 3 == 2:  # a sorted row: each owner's keys sit in a few chunks (sub-slot overflow)
            x32[0] = np.sort(x32[0])
        _check(x32, dn, k, b, kb)


def test_xb_first_call_inside_graph_capture(tmp_path):
    """A fresh process whose first exchange call (several batches: the side
    stream and its events are created lazily) happens inside CUDA graph
    capture: capture succeeds and the replay equals an eager call."""
    import subprocess
    import sys
    script = tmp_path / "cap.py"
    script.write_text(
        "import os, sys, torch\n"
        "sys.path.insert(0, os.getcwd())\n"
        "os.environ['BTK_XB_ROWS'] = '2'\n"
        "import paper_2412_04358_b200 as btk\n"
        "x = torch.randn(5, 262144, device='cuda').to(torch.bfloat16)\n"
        "op = btk.ApproxTopK(5, 262144, 20000, btk.BucketScheme(16384, 2), dtype=torch.bfloat16, device='cuda')\n"
        "s = torch.cuda.Stream()\n"
        "g = torch.cuda.CUDAGraph()\n"
        "with torch.cuda.stream(s):\n"
        "    with torch.cuda.graph(g, stream=s):\n"
        "        op.launch(x)\n"
        "g.replay()\n"
        "torch.cuda.synchronize()\n"
        "r = btk.approx_topk(x, 20000, btk.BucketScheme(16384, 2))\n"
        "assert torch.equal(op.indices, r.indices) and torch.equal(op.values, r.values)\n"
        "print('ok')\n")
    out = subprocess.run([sys.executable, str(script)], capture_output=True, text=True, timeout=300,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
