"""Reference-side binding: the module a `bucketed_topk` maintainer adds
(as `bucketed_topk/_b200.py`) to run the hot path on a B200.

It binds the C ABI of libbtk.so (include/btk.h) with ctypes — plain
pointers, sizes and status codes; torch only allocates device memory —
and returns the REFERENCE's own result types.  Nothing is rounded: the
reference computes in float64 (`exact._as_matrix`, exact.py:87-96) and so
does this binding (BTK_F64, 128-bit composite keys), so every result is
bit-identical to the reference's on the same input, including ties, the
sign of zero and subnormals.

    import bucketed_topk
    from integration import bucketed_topk_b200 as b200
    b200.install(bucketed_topk)        # opt-in: reference callers now run on the GPU
    ...
    b200.uninstall(bucketed_topk)

`install` rebinds approx_topk / stage1 / exact_topk_oracle /
priority_queue_topk / topk_with_indices in the package and in the modules
that imported them by name (cli.py, bench.py, recall.py), so
`cli.cmd_run` (cli.py:256), `bench.time_selection` (bench.py:126) and
`recall.monte_carlo_recall` (recall.py:262) call the GPU unchanged.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BTK_LIB") or os.path.join(os.path.dirname(_HERE), "paper_2412_04358_b200",
                                                     "libbtk.so")

_i64, _vp, _sz, _i = ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
BTK_F64 = 3
_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(LIB_PATH)
        lib.btk_workspace_bytes.restype = _sz
        lib.btk_workspace_bytes.argtypes = [_i64] * 5 + [_i, _i]
        lib.btk_approx_topk.restype = _i
        lib.btk_approx_topk.argtypes = [_vp, _i64, _i] + [_i64] * 5 + [_i, _vp, _vp, _vp, _sz, _vp, _vp]
        lib.btk_stage1_workspace_bytes.restype = _sz
        lib.btk_stage1_workspace_bytes.argtypes = [_i64] * 4 + [_i, _i]
        lib.btk_stage1.restype = _i
        lib.btk_stage1.argtypes = [_vp, _i64, _i] + [_i64] * 4 + [_i, _vp, _vp, _vp, _sz, _vp, _vp]
        lib.btk_stage1_count.restype = _i64
        lib.btk_stage1_count.argtypes = [_i64, _i64, _i64, _i]
        lib.btk_exact_workspace_bytes.restype = _sz
        lib.btk_exact_workspace_bytes.argtypes = [_i64] * 3 + [_i]
        lib.btk_exact_topk.restype = _i
        lib.btk_exact_topk.argtypes = [_vp, _i64, _i] + [_i64] * 3 + [_vp, _vp, _vp, _sz, _vp, _vp]
        lib.btk_topk_with_indices_workspace_bytes.restype = _sz
        lib.btk_topk_with_indices_workspace_bytes.argtypes = [_i64] * 3 + [_i]
        lib.btk_topk_with_indices.restype = _i
        lib.btk_topk_with_indices.argtypes = [_vp, _vp, _i] + [_i64] * 3 + [_vp, _vp, _vp, _sz, _vp, _vp]
        lib.btk_error_code.restype = ctypes.c_char_p
        lib.btk_error_code.argtypes = [_i]
        lib.btk_error_string.restype = ctypes.c_char_p
        lib.btk_error_string.argtypes = [_i]
        _lib = lib
    return _lib


def _ref():
    import bucketed_topk.approx as approx
    import bucketed_topk.core as core
    import bucketed_topk.exact as exact
    return approx, core, exact


def _as_matrix(scores):
    # reference exact.py:87-96, verbatim semantics: float64, 1-D -> 1 row,
    # shape and finiteness checked on the host before any device work
    _, _, exact = _ref()
    return exact._as_matrix(scores)


class _Dev:
    """Device buffers for one call (torch supplies memory and the stream)."""

    def __init__(self):
        import torch
        self.torch = torch
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.stream = torch.cuda.current_stream(self.dev).cuda_stream

    def put(self, a):
        return self.torch.from_numpy(np.ascontiguousarray(a)).to(self.dev)

    def empty(self, shape, dtype):
        return self.torch.empty(shape, dtype=dtype, device=self.dev)

    def ws(self, nbytes):
        return self.torch.empty(max(int(nbytes), 1), dtype=self.torch.uint8, device=self.dev)

    def flag(self):
        return self.torch.zeros(1, dtype=self.torch.int32, device=self.dev)


def _check(st, flag):
    _, core, _ = _ref()
    lib = _load()
    if st:
        code = lib.btk_error_code(st).decode()
        msg = lib.btk_error_string(st).decode()
        if 1 <= st <= 8:
            raise core.ConfigError(code, msg)
        raise RuntimeError(f"libbtk: {code}: {msg}")
    if int(flag.item()) & 1:
        raise core.NonFiniteInputError("scores contain NaN or infinity")


def _layout(scheme):
    return 0 if scheme.assignment.value == "interleaved" else 1


def approx_topk(scores, k, scheme, mode=None, workers=1):
    """Drop-in for bucketed_topk.approx.approx_topk (approx.py:245-282)."""
    approx, core, exact = _ref()
    a = _as_matrix(scores)
    m, n = a.shape
    core.check_parameters(m, n, k, scheme.b, scheme.k_b)
    if mode is not None and not isinstance(mode, (approx.PerBucket, approx.ChunkedMerge)):
        raise TypeError(f"unknown execution mode {mode!r}")
    lib, d = _load(), _Dev()
    x = d.put(a)
    vals = d.empty((m, k), d.torch.float64)
    idx = d.empty((m, k), d.torch.int64)
    flag = d.flag()
    wsb = lib.btk_workspace_bytes(m, n, k, scheme.b, scheme.k_b, BTK_F64, _layout(scheme))
    ws = d.ws(wsb)
    st = lib.btk_approx_topk(x.data_ptr(), n, BTK_F64, m, n, k, scheme.b, scheme.k_b, _layout(scheme),
                             vals.data_ptr(), idx.data_ptr(), ws.data_ptr(), wsb, flag.data_ptr(), d.stream)
    _check(st, flag)
    return exact.TopKResult(values=vals.cpu().numpy(), indices=idx.cpu().numpy())


def stage1(scores, scheme, mode=None):
    """Drop-in for bucketed_topk.approx.stage1 (approx.py:208-242)."""
    approx, core, exact = _ref()
    a = _as_matrix(scores)
    m, n = a.shape
    b, kb = scheme.b, scheme.k_b
    if not isinstance(b, (int, np.integer)) or not 1 <= b <= n:
        raise core.ConfigError("b_gt_n", f"b must be in 1..n (b={b}, n={n})")
    cap = core.max_bucket_size(n, b)
    if not isinstance(kb, (int, np.integer)) or not 1 <= kb <= cap:
        raise core.ConfigError("kb_range", f"k_b out of range (k_b={kb}, allowed 1..ceil(n/b)={cap})")
    lib, d = _load(), _Dev()
    lay = _layout(scheme)
    C = lib.btk_stage1_count(n, b, kb, lay)
    x = d.put(a)
    vals = d.empty((m, C), d.torch.float64)
    idx = d.empty((m, C), d.torch.int64)
    flag = d.flag()
    wsb = lib.btk_stage1_workspace_bytes(m, n, b, kb, BTK_F64, lay)
    ws = d.ws(wsb)
    st = lib.btk_stage1(x.data_ptr(), n, BTK_F64, m, n, b, kb, lay, vals.data_ptr(), idx.data_ptr(),
                        ws.data_ptr(), wsb, flag.data_ptr(), d.stream)
    _check(st, flag)
    per_bucket = np.minimum(core.bucket_sizes(n, b, scheme.assignment), kb)
    return approx.Stage1Candidates(values=vals.cpu().numpy(), indices=idx.cpu().numpy(),
                                   per_bucket=per_bucket)


def exact_topk_oracle(scores, k, workers=1):
    """Drop-in for bucketed_topk.exact.exact_topk_oracle (exact.py:162-173)."""
    _, _, exact = _ref()
    a = _as_matrix(scores)
    m, n = a.shape
    exact._check_k(k, n)
    lib, d = _load(), _Dev()
    x = d.put(a)
    vals = d.empty((m, k), d.torch.float64)
    idx = d.empty((m, k), d.torch.int64)
    flag = d.flag()
    wsb = lib.btk_exact_workspace_bytes(m, n, k, BTK_F64)
    ws = d.ws(wsb)
    st = lib.btk_exact_topk(x.data_ptr(), n, BTK_F64, m, n, k, vals.data_ptr(), idx.data_ptr(),
                            ws.data_ptr(), wsb, flag.data_ptr(), d.stream)
    _check(st, flag)
    return exact.TopKResult(values=vals.cpu().numpy(), indices=idx.cpu().numpy())


def topk_with_indices(values, indices, k):
    """Drop-in for bucketed_topk.exact.topk_with_indices (exact.py:142-159)."""
    _, core, exact = _ref()
    v = np.asarray(values, dtype=np.float64)
    i = np.asarray(indices, dtype=np.int64)
    if v.ndim == 1:
        v, i = v[None], i[None]
    if v.shape != i.shape:
        raise ValueError("values and indices must have matching shapes")
    m, c = v.shape
    exact._check_k(k, c)
    lib, d = _load(), _Dev()
    xv, xi = d.put(v), d.put(i)
    ov = d.empty((m, k), d.torch.float64)
    oi = d.empty((m, k), d.torch.int64)
    flag = d.flag()
    wsb = lib.btk_topk_with_indices_workspace_bytes(m, c, k, BTK_F64)
    ws = d.ws(wsb)
    st = lib.btk_topk_with_indices(xv.data_ptr(), xi.data_ptr(), BTK_F64, m, c, k, ov.data_ptr(),
                                   oi.data_ptr(), ws.data_ptr(), wsb, flag.data_ptr(), d.stream)
    _check(st, flag)
    if int(flag.item()) & 2:
        raise ValueError("carried labels must lie in [0, 2**31 - 1] on the GPU path")
    return exact.TopKResult(values=ov.cpu().numpy(), indices=oi.cpu().numpy())


def priority_queue_topk(scores, k, workers=1):
    """Same contract as exact_topk_oracle (exact.py:176-220)."""
    return exact_topk_oracle(scores, k, workers)


_NAMES = ("approx_topk", "stage1", "exact_topk_oracle", "priority_queue_topk", "topk_with_indices")
_saved = {}


def install(pkg) -> None:
    """Opt-in: rebind the hot-path names in the reference package and in its
    modules that imported them (cli, bench, recall, approx)."""
    import importlib

    mods = [pkg] + [importlib.import_module(f"{pkg.__name__}.{s}")
                    for s in ("approx", "exact", "cli", "bench", "recall")]
    for mod in mods:
        for name in _NAMES:
            if hasattr(mod, name):
                _saved.setdefault((mod.__name__, name), getattr(mod, name))
                setattr(mod, name, globals()[name])


def uninstall(pkg) -> None:
    import sys

    for (modname, name), fn in list(_saved.items()):
        if modname in sys.modules:
            setattr(sys.modules[modname], name, fn)
    _saved.clear()
