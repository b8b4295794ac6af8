"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/btk.h declares, and its host-side logic (validation codes,
candidate counts, byte formula) matches the reference's golden values.
No compute calls here (no GPU in the build container)."""

import os
import re

import numpy as np
import pytest

from paper_2412_04358_b200 import _lib
from paper_2412_04358_b200.core import Assignment, stage1_candidate_count
from tests.golden_io import load

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(REPO, "include", "btk.h")).read()
    return sorted(set(re.findall(r"\b(btk_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), "ctypes table out of sync with btk.h"


def test_c_validate_matches_reference_codes():
    lib = _lib.load()
    z = load("validation.npz")
    for p, code in zip(z["params"], z["codes"]):
        st = lib.btk_validate(*(int(v) for v in p))
        assert _lib.error_code(st) == str(code), (p, code)


@pytest.mark.parametrize("layout", [0, 1])
def test_c_stage1_count(layout):
    lib = _lib.load()
    asg = Assignment.INTERLEAVED if layout == 0 else Assignment.CONTIGUOUS
    for n in range(1, 60):
        for b in range(1, n + 1):
            for kb in range(1, -(-n // b) + 1):
                assert lib.btk_stage1_count(n, b, kb, layout) == stage1_candidate_count(n, b, kb, asg)


def test_c_min_bytes_known_answer():
    # reference test_bench.py:81-88
    assert _lib.load().btk_min_bytes(128, 2**20, 64, 4, 8) == 536_969_216


def test_error_strings_cover_codes():
    for s in range(0, 15):
        assert _lib.error_code(s) != "unknown"
        assert _lib.error_string(s)


# (m, n, k, b, kb, dtype, fused?, launches per call) for the BASELINE configs
_PLANS = [
    (128, 65536, 64, 64, 1, _lib.BTK_F32, 1, 1),            # cfg1: cluster kernel
    (128, 65536, 16384, 8192, 2, _lib.BTK_F32, 1, 1),       # cfg2: wide kernel
    (128, 65536, 16384, 2048, 8, _lib.BTK_F32, 1, 1),
    (128, 1 << 20, 256, 512, 1, _lib.BTK_BF16, 1, 1),       # cfg3
    (4096, 32768, 512, 512, 1, _lib.BTK_BF16, 1, 1),        # cfg4: warp-per-row kernel
    # cfg5: batched exchange (split, 56 batches of 148 rows x (partition, sort), fallback kernel)
    (8192, 1 << 20, 65536, 65536, 2, _lib.BTK_BF16, 1, 114),
]


@pytest.mark.parametrize("plan", _PLANS, ids=lambda p: f"m{p[0]}-n{p[1]}-k{p[2]}-b{p[3]}-kb{p[4]}")
def test_launch_planner_host_side(plan):
    """The host-side planner (no GPU needed) picks the fused single-launch
    path for cfg1-4 and the exchange pipeline (batched partition + owner sorts, plus its
    fallback K2) for cfg5, and sizes the workspace for the path that runs."""
    m, n, k, b, kb, dt, fused, launches = plan
    lib = _lib.load()
    assert lib.btk_uses_fused_path(m, n, k, b, kb, dt, _lib.BTK_INTERLEAVED, n) == fused
    assert lib.btk_launch_count(m, n, k, b, kb, dt, _lib.BTK_INTERLEAVED, n) == launches
    # sized for the generic path too (the fused path's eligibility also
    # depends on the input pointer's alignment, unknown here)
    ws = lib.btk_workspace_bytes(m, n, k, b, kb, dt, _lib.BTK_INTERLEAVED)
    assert ws >= (0 if fused else m * b * kb * 8)
    # contiguous layout always takes the generic path
    assert lib.btk_uses_fused_path(m, n, k, b, kb, dt, _lib.BTK_CONTIGUOUS, n) == 0
    # a misaligned row stride (not 16-byte multiple) drops out of the fused envelope
    assert lib.btk_uses_fused_path(m, n, k, b, kb, dt, _lib.BTK_INTERLEAVED, n + 1) == 0


@pytest.mark.parametrize("m,launches", [(1, 4), (148, 4), (149, 6), (300, 8), (8192, 114)])
def test_exchange_launch_count_per_batch(m, launches, monkeypatch):
    """The batched exchange: split + (partition, sort) per batch of <= 148
    rows + the fallback kernel; BTK_XB=0 (cluster kernel): 2 launches; the
    workspace is sized for the row cap whatever BTK_XB_ROWS says."""
    lib = _lib.load()
    args = (m, 1 << 20, 65536, 65536, 2, _lib.BTK_BF16, _lib.BTK_INTERLEAVED, 1 << 20)
    assert lib.btk_launch_count(*args) == launches
    ws = lib.btk_plan_workspace_bytes(256, 1 << 20, _lib.BTK_BF16, m, 1 << 20, 65536, 65536, 2,
                                      _lib.BTK_INTERLEAVED)
    monkeypatch.setenv("BTK_XB_ROWS", "2")
    assert lib.btk_plan_workspace_bytes(256, 1 << 20, _lib.BTK_BF16, m, 1 << 20, 65536, 65536, 2,
                                        _lib.BTK_INTERLEAVED) == ws
    assert lib.btk_launch_count(*args) == 2 + 2 * -(-m // 2)
    monkeypatch.setenv("BTK_XB", "0")
    assert lib.btk_launch_count(*args) == 2


@pytest.mark.parametrize("s", ["1", "2", "4", "8"])
def test_planner_cluster_overrides_stay_valid(s, monkeypatch):
    monkeypatch.setenv("BTK_S", s)
    monkeypatch.setenv("BTK_ROWS", "0")
    lib = _lib.load()
    for (m, n, k, b, kb, dt) in [(3, 65536, 64, 64, 1, _lib.BTK_F32), (2, 131072, 256, 1024, 1, _lib.BTK_BF16)]:
        assert lib.btk_uses_fused_path(m, n, k, b, kb, dt, _lib.BTK_INTERLEAVED, n) == 1
