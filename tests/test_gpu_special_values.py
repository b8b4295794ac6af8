"""Subnormals and signed zeros through EVERY kernel family and launch shape.

The ordering contract (reference exact.py:130-139, approx.py:151-162):
value descending with IEEE compares (-0.0 == +0.0, subnormals ordered
exactly), ties by lower index, output values are the input bits (sign of
zero kept).  Inputs come from tests/special_inputs.py: bit patterns built
in the target dtype with the k-th boundary inside the subnormal / zero
band, so the fused kernels' float compares (Queue::push), the packed
HSET2 bf16/fp16 scanner and the 64-bit composite keys all see them.
"""

import numpy as np
import pytest
import torch

import paper_2412_04358_b200 as btk
from paper_2412_04358_b200 import _lib
from oracle import bucketed_oracle as O
from tests.special_inputs import TORCH, has_subnormal, special, to_dtype

pytestmark = pytest.mark.gpu

I = btk.Assignment.INTERLEAVED
_DTC = {"f32": _lib.BTK_F32, "bf16": _lib.BTK_BF16, "f16": _lib.BTK_F16}


def _bits(t):
    t = t.detach().cpu()
    return t.view(torch.int32 if t.dtype == torch.float32 else torch.int16).numpy()


def _want_bits(v64, dn):
    return _bits(torch.from_numpy(np.asarray(v64, np.float64)).to(TORCH[dn]))


def family(m, n, k, b, kb, dn, layout=_lib.BTK_INTERLEAVED):
    return _lib.load().btk_kernel_family(m, n, k, b, kb, _DTC[dn], layout, n)


def check(x32, dn, k, b, kb, asg=I):
    wv, wi = O.approx_topk(x32, k, b, kb, "interleaved" if asg is I else "contiguous")
    x = to_dtype(x32, dn).cuda()
    r = btk.approx_topk(x, k, btk.BucketScheme(b, kb, asg))
    np.testing.assert_array_equal(r.indices.cpu().numpy(), wi)
    np.testing.assert_array_equal(_bits(r.values), _want_bits(wv, dn))
    return r


# (m, n, k, b, kb): narrow (cluster) / rows / wide / s1_vec pool shapes
CASES = [
    (3, 65536, 64, 64, 1),        # cfg1 shape (narrow, S=2)
    (2, 32768, 512, 512, 1),      # cfg4 shape (narrow or rows)
    (3, 40000, 512, 128, 4),
    (2, 33000, 256, 64, 8),       # ragged final view-row
    (4, 8192 + 64, 100, 64, 2),
    (2, 131072, 256, 1024, 1),
    (2, 65536, 8192, 4096, 2),    # wide (f32 and 16-bit)
    (2, 32768, 4096, 2048, 2),    # wide (f32), narrow (16-bit)
]
KINDS = ("subnormal", "subnormal_ties", "pm0")
_SHAPE_ENVS = [{"BTK_ROWS": "1"}, {"BTK_ROWS": "0", "BTK_S": "1"}, {"BTK_ROWS": "0", "BTK_S": "2"},
               {"BTK_ROWS": "0", "BTK_S": "4"}, {"BTK_ROWS": "0", "BTK_S": "8"},
               {"BTK_ROWS": "0", "BTK_S": "2", "BTK_STAGE_KB": "8", "BTK_NS": "3"}]


@pytest.mark.parametrize("env", _SHAPE_ENVS, ids=lambda e: "-".join(f"{k[4:]}{v}" for k, v in e.items()))
@pytest.mark.parametrize("dn", ["f32", "bf16", "f16"])
def test_fused_shapes_special_values(env, dn, monkeypatch):
    for k_, v_ in env.items():
        monkeypatch.setenv(k_, v_)
    rng = np.random.default_rng(4242)
    fams = set()
    for m, n, k, b, kb in CASES:
        if dn != "f32" and kb == 8:
            continue  # 16-bit k_b = 8 is outside the fused envelope (V * k_b > 32)
        fams.add(family(m, n, k, b, kb, dn))
        for kind in KINDS:
            x32 = special(rng, kind, m, n, dn)
            if kind != "pm0":
                assert has_subnormal(x32, dn)
            check(x32, dn, k, b, kb)
    assert fams <= {1, 2, 3}, fams  # every case stayed on a fused kernel
    if env.get("BTK_ROWS") == "1":
        assert 3 in fams, fams  # the warp-per-row kernel really ran


@pytest.mark.parametrize("dn", ["f32", "bf16", "f16"])
def test_every_family_special_values(dn):
    """One case per kernel family (asserted through btk_kernel_family)."""
    rng = np.random.default_rng(99)
    cases = {
        1: (3, 65536, 64, 64, 1),          # narrow
        2: (2, 65536, 8192, 4096, 2),      # wide
        3: (1200, 2048, 64, 64, 1),        # rows (m >= 8 * #SMs)
        7: (2, 131072, 16384, 16384, 2),   # s1_vec pool + histogram-chunked Stage 2 (fp32)
        8: (2, 131072, 16384, 16384, 2),   # cluster exchange (16-bit; same shape)
        0: (2, 20000, 700, 999, 3),        # generic (b % V != 0)
        5: (2, 30000, 300, 1, 300),        # materialise (b == 1)
    }
    for fam, (m, n, k, b, kb) in cases.items():
        if (fam == 7) != (dn == "f32") and fam in (7, 8):
            continue  # large pools: fp32 -> chunked pool, 16-bit -> cluster exchange
        assert family(m, n, k, b, kb, dn) == fam, (fam, dn)
        for kind in KINDS:
            check(special(rng, kind, m, n, dn), dn, k, b, kb)
    # contiguous layout (warp-per-bucket family)
    m, n, k, b, kb = 2, 20000, 512, 256, 2
    assert family(m, n, k, b, kb, dn, _lib.BTK_CONTIGUOUS) == _lib.BTK_FAM_CONTIG
    for kind in KINDS:
        check(special(rng, kind, m, n, dn), dn, k, b, kb, btk.Assignment.CONTIGUOUS)


@pytest.mark.parametrize("chunked", ["1", "0"])
@pytest.mark.parametrize("dn", ["f32", "bf16", "f16"])
def test_long_pool_special_values(dn, chunked, monkeypatch):
    """Pool > 16384 without the cluster exchange (BTK_XC=0): the
    histogram-chunked Stage 2 (its per-row radix-select fallback for
    tie-heavy rows included), and with BTK_POOL_CHUNKED=0 the
    select/compact + global LSD path."""
    monkeypatch.setenv("BTK_POOL_CHUNKED", chunked)
    monkeypatch.setenv("BTK_XC", "0")
    rng = np.random.default_rng(5)
    for (m, n, k, b, kb) in [(2, 262144, 20000, 16384, 2), (3, 131072, 12000, 16384, 2)]:
        assert family(m, n, k, b, kb, dn) == (7 if chunked == "1" else 4)
        for kind in ("subnormal", "pm0", "subnormal_ties"):
            check(special(rng, kind, m, n, dn), dn, k, b, kb)
        # mixed rows: tie-heavy rows take the fallback, normal rows the chunks
        x32 = special(rng, "pm0", m, n, dn)
        x32[1] = torch.from_numpy(rng.standard_normal(n, dtype=np.float32)).to(TORCH[dn]).float().numpy()
        check(x32, dn, k, b, kb)


@pytest.mark.parametrize("dn", ["f32", "bf16", "f16"])
def test_stage1_and_exact_special_values(dn):
    """stage1() candidates and exact_topk_oracle on the same inputs."""
    rng = np.random.default_rng(6)
    for (m, n, b, kb) in [(2, 65536, 64, 1), (2, 65536, 4096, 2), (3, 5000, 50, 3)]:
        x32 = special(rng, "subnormal_ties", m, n, dn)
        x = to_dtype(x32, dn).cuda()
        c = btk.stage1(x, btk.BucketScheme(b, kb, I))
        wv, wi, _ = O.stage1(O.as_matrix(x32), b, kb, "interleaved")
        np.testing.assert_array_equal(c.indices.cpu().numpy(), wi)
        np.testing.assert_array_equal(_bits(c.values), _want_bits(wv, dn))
        e = btk.exact_topk_oracle(x, 100)
        ev, ei = O.exact_topk(x32, 100)
        np.testing.assert_array_equal(e.indices.cpu().numpy(), ei)
        np.testing.assert_array_equal(_bits(e.values), _want_bits(ev, dn))
