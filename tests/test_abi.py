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
