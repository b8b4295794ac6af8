"""ctypes binding of libbtk.so (include/btk.h).

This is the drop-in boundary: plain pointers and sizes in, status codes
out.  There is no fallback: if the library is missing the import of any
compute entry point raises, loudly.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# BTK_LIB overrides the library file (development A/B runs of two builds)
LIB_PATH = os.environ.get("BTK_LIB") or os.path.join(_HERE, "libbtk.so")

BTK_F32, BTK_BF16, BTK_F16, BTK_F64 = 0, 1, 2, 3
(BTK_FAM_GENERIC, BTK_FAM_NARROW, BTK_FAM_WIDE, BTK_FAM_ROWS, BTK_FAM_VEC_POOL, BTK_FAM_MATERIALIZE,
 BTK_FAM_F64, BTK_FAM_POOL_CHUNKED, BTK_FAM_XCHG, BTK_FAM_CONTIG) = range(10)
BTK_INTERLEAVED, BTK_CONTIGUOUS = 0, 1
BTK_INPUT_READY = 1

_i64, _sz, _vp, _i = ctypes.c_int64, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_int

# name -> (restype, argtypes); every symbol include/btk.h declares.
SIGNATURES = {
    "btk_validate": (_i, [_i64] * 5),
    "btk_stage1_validate": (_i, [_i64] * 3),
    "btk_stage1_count": (_i64, [_i64, _i64, _i64, _i]),
    "btk_workspace_bytes": (_sz, [_i64] * 5 + [_i, _i]),
    "btk_plan_workspace_bytes": (_sz, [_vp, _i64, _i] + [_i64] * 5 + [_i]),
    "btk_approx_topk": (_i, [_vp, _i64, _i] + [_i64] * 5 + [_i, _vp, _vp, _vp, _sz, _vp, _vp]),
    "btk_approx_topk_flags": (_i, [_vp, _i64, _i] + [_i64] * 5 + [_i, _vp, _vp, _vp, _sz, _vp,
                                                               ctypes.c_uint32, _vp]),
    "btk_stage1_workspace_bytes": (_sz, [_i64] * 4 + [_i, _i]),
    "btk_stage1": (_i, [_vp, _i64, _i] + [_i64] * 4 + [_i, _vp, _vp, _vp, _sz, _vp, _vp]),
    "btk_exact_workspace_bytes": (_sz, [_i64] * 3 + [_i]),
    "btk_exact_topk": (_i, [_vp, _i64, _i] + [_i64] * 3 + [_vp, _vp, _vp, _sz, _vp, _vp]),
    "btk_topk_with_indices_workspace_bytes": (_sz, [_i64] * 3 + [_i]),
    "btk_topk_with_indices": (_i, [_vp, _vp, _i] + [_i64] * 3 + [_vp, _vp, _vp, _sz, _vp, _vp]),
    "btk_recall_hits": (_i, [_vp, _i64, _vp, _i64, _i64, _i64, _vp, _vp]),
    "btk_min_bytes": (_i64, [_i64] * 5),
    "btk_uses_fused_path": (_i, [_i64] * 5 + [_i, _i, _i64]),
    "btk_launch_count": (_i, [_i64] * 5 + [_i, _i, _i64]),
    "btk_kernel_family": (_i, [_i64] * 5 + [_i, _i, _i64]),
    "btk_error_code": (ctypes.c_char_p, [_i]),
    "btk_error_string": (ctypes.c_char_p, [_i]),
    "btk_last_cuda_error": (_i, []),
    "btk_version": (ctypes.c_char_p, []),
}

_lock = threading.Lock()
_lib = None


class LibraryMissing(RuntimeError):
    pass


def load() -> ctypes.CDLL:
    """Load (once) and type the C-ABI library.  Raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise LibraryMissing(
                    f"{LIB_PATH} not built; run `python -m paper_2412_04358_b200.build` "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def error_code(status: int) -> str:
    return load().btk_error_code(status).decode()


def error_string(status: int) -> str:
    return load().btk_error_string(status).decode()
