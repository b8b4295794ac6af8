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
