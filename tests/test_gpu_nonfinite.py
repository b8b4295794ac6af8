"""Every kernel family flags NaN / +inf / -inf anywhere in its input
(reference exact.py:87-96 `_as_matrix` rejects non-finite scores), including
positions that never become candidates (a -inf is never a bucket maximum),
and completes without faults on such rows (check_finite=False)."""

import pytest
import torch

import paper_2412_04358_b200 as btk
from paper_2412_04358_b200 import _lib

pytestmark = pytest.mark.gpu

I, Cg = btk.Assignment.INTERLEAVED, btk.Assignment.CONTIGUOUS
_DTC = {torch.float32: _lib.BTK_F32, torch.bfloat16: _lib.BTK_BF16, torch.float16: _lib.BTK_F16}

# (m, n, k, b, kb, dtype, assignment, env): one shape per family
CASES = [
    (3, 65536, 64, 64, 1, torch.float32, I, {}),                       # fused_narrow
    (2, 65536, 16384, 8192, 2, torch.float32, I, {}),                  # fused_wide
    (1200, 2048, 64, 64, 1, torch.bfloat16, I, {}),                    # fused_rows
    (3, 262144, 20000, 16384, 2, torch.bfloat16, I, {}),               # batched exchange
    (3, 262144, 20000, 16384, 2, torch.float16, I, {"BTK_XB": "0"}),   # cluster exchange
    (2, 262144, 20000, 16384, 2, torch.float32, I, {}),                # s1_vec + chunked pool
    (2, 131072, 256, 512, 1, torch.bfloat16, Cg, {}),                  # s1_contig
    (2, 20000, 700, 999, 3, torch.float32, I, {}),                     # generic
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[5]}-m{c[0]}-n{c[1]}-k{c[2]}-b{c[3]}-kb{c[4]}-{c[6].name}-{'_'.join(c[7])}")
def test_nonfinite_flagged_in_every_family(case, monkeypatch):
    m, n, k, b, kb, dt, asg, env = case
    for key, v in env.items():
        monkeypatch.setenv(key, v)
    lib = _lib.load()
    fam = lib.btk_kernel_family(m, n, k, b, kb, _DTC[dt], 0 if asg == I else 1, n)
    g = torch.Generator(device="cuda").manual_seed(7)
    base = torch.randn(m, n, device="cuda", generator=g).to(dt)
    for bad in (float("nan"), float("inf"), float("-inf")):
        x = base.clone()
        x[m - 1, (n * 7) // 11] = bad
        with pytest.raises(btk.NonFiniteInputError):
            btk.approx_topk(x, k, btk.BucketScheme(b, kb, asg))
        r = btk.approx_topk(x, k, btk.BucketScheme(b, kb, asg), check_finite=False)
        torch.cuda.synchronize()
        assert tuple(r.indices.shape) == (m, k), fam
    # and the finite input passes
    btk.approx_topk(base, k, btk.BucketScheme(b, kb, asg))
