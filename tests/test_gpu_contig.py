"""Contiguous bucket layout through the warp-per-bucket Stage 1
(s1_contig, family BTK_FAM_CONTIG) + K2, against the oracle: aligned and
unaligned slices (ragged b that does not divide n), every k_b it serves,
every dtype, ties and signed zeros / subnormals.
Reference: core.py:124-147 (contiguous buckets), approx.py:121-124."""

import numpy as np
import pytest
import torch

import paper_2412_04358_b200 as btk
from paper_2412_04358_b200 import _lib
from oracle import bucketed_oracle as O
from tests.special_inputs import TORCH, special, to_dtype

pytestmark = pytest.mark.gpu
C = btk.Assignment.CONTIGUOUS
_DTC = {"f32": _lib.BTK_F32, "bf16": _lib.BTK_BF16, "f16": _lib.BTK_F16}


def _bits(t):
    t = t.detach().cpu()
    return t.view(torch.int32 if t.dtype == torch.float32 else torch.int16).numpy()


def _check(x32, dn, k, b, kb):
    x = to_dtype(x32, dn).cuda()
    r = btk.approx_topk(x, k, btk.BucketScheme(b, kb, C))
    wv, wi = O.approx_topk(x32, k, b, kb, "contiguous")
    np.testing.assert_array_equal(r.indices.cpu().numpy(), wi)
    np.testing.assert_array_equal(_bits(r.values), _bits(torch.from_numpy(np.asarray(wv, np.float64)).to(TORCH[dn])))
    s = btk.stage1(x, btk.BucketScheme(b, kb, C))
    sv, si, _ = O.stage1(O.as_matrix(x32), b, kb, "contiguous")
    np.testing.assert_array_equal(s.indices.cpu().numpy(), si)


SHAPES = [
    (3, 1 << 16, 256, 512, 1),      # aligned slices of 128 elements
    (2, 1 << 17, 512, 256, 2),
    (2, 100000, 300, 97, 4),        # ragged: slices of 1030/1031, unaligned starts
    (3, 33000, 400, 50, 8),
    (2, 4096, 64, 4096, 1),         # one element per bucket
    (2, 1000, 30, 7, 5),
]


@pytest.mark.parametrize("dn", ["f32", "bf16", "f16"])
def test_contig_normal_ties(dn):
    rng = np.random.default_rng(21)
    for (m, n, k, b, kb) in SHAPES:
        assert _lib.load().btk_kernel_family(m, n, k, b, kb, _DTC[dn], _lib.BTK_CONTIGUOUS, n) == _lib.BTK_FAM_CONTIG
        x32 = torch.from_numpy(rng.standard_normal((m, n), dtype=np.float32)).to(TORCH[dn]).float().numpy()
        _check(x32, dn, k, b, kb)
        _check(np.round(x32 * 2) / 2, dn, k, b, kb)


@pytest.mark.parametrize("dn", ["f32", "bf16", "f16"])
def test_contig_special_values(dn):
    rng = np.random.default_rng(22)
    for (m, n, k, b, kb) in SHAPES[:4]:
        for kind in ("subnormal", "subnormal_ties", "pm0"):
            _check(special(rng, kind, m, n, dn), dn, k, b, kb)


def test_contig_cfg3_shape_full_rows():
    """BASELINE cfg3 shape with contiguous buckets: every row against the
    oracle on a row subset, and equal to the generic path on all rows."""
    m, n, k, b, kb = 128, 1 << 20, 256, 512, 1
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn((m, n), generator=g, device="cuda").to(torch.bfloat16)
    r = btk.approx_topk(x, k, btk.BucketScheme(b, kb, C))
    rows = [0, 17, 127]
    wv, wi = O.approx_topk(x[rows].float().cpu().numpy(), k, b, kb, "contiguous")
    np.testing.assert_array_equal(r.indices[rows].cpu().numpy(), wi)


def test_exact_and_large_kb_select_without_materialising():
    """exact_topk_oracle (b = 1) and k_b > 16 stage 1 select straight from
    the scores: the workspace is O(m*k), not O(m*n) (a 8192 x 2^20 exact
    top-65536 needs 12.9 GB instead of 68.7 GB), and the results are the
    oracle's (reference exact.py:162-173, approx.py:142-164)."""
    lib = _lib.load()
    assert lib.btk_exact_workspace_bytes(8192, 1 << 20, 65536, _lib.BTK_BF16) < 8192 * (1 << 20) * 8 // 5
    assert lib.btk_exact_workspace_bytes(128, 65536, 64, _lib.BTK_F32) <= 128 * 64 * 8 + 512
    rng = np.random.default_rng(31)
    x32 = torch.from_numpy(rng.standard_normal((3, 1 << 20), dtype=np.float32)).to(torch.bfloat16).float().numpy()
    x32[1, ::3] = 0.25  # heavy ties at the boundary
    x = to_dtype(x32, "bf16").cuda()
    for k in (37, 20000):
        e = btk.exact_topk_oracle(x, k)
        wv, wi = O.exact_topk(x32, k)
        np.testing.assert_array_equal(e.indices.cpu().numpy(), wi)
    for (n, b, kb, asg) in [(50000, 100, 300, "interleaved"), (50000, 100, 300, "contiguous"), (70000, 7, 17, "interleaved")]:
        xs = rng.standard_normal((2, n), dtype=np.float32)
        xs[0, ::4] = -0.0
        A = btk.Assignment.from_string(asg)
        k = min(b * kb, 1000)
        r = btk.approx_topk(torch.from_numpy(xs).cuda(), k, btk.BucketScheme(b, kb, A))
        wv, wi = O.approx_topk(xs, k, b, kb, asg)
        np.testing.assert_array_equal(r.indices.cpu().numpy(), wi)
        s = btk.stage1(torch.from_numpy(xs).cuda(), btk.BucketScheme(b, kb, A))
        sv, si, _ = O.stage1(O.as_matrix(xs), b, kb, asg)
        np.testing.assert_array_equal(s.indices.cpu().numpy(), si)
