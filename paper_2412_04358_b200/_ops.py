"""Tensor plumbing between the Python API and the C ABI.

torch supplies device memory, streams and the caching allocator; every
compute step is a libbtk.so kernel.  Inputs are CUDA tensors, or NumPy /
CPU tensors / lists, which are copied to the current CUDA device first
(the reference's callers pass NumPy float64 arrays: float64 has its own
exact GPU path, nothing is rounded).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .core import ConfigError, NonFiniteInputError

_DTYPES = {torch.float32: _lib.BTK_F32, torch.bfloat16: _lib.BTK_BF16, torch.float16: _lib.BTK_F16,
           torch.float64: _lib.BTK_F64}

# status codes that correspond to reference ConfigError codes
_CONFIG_CODES = {1, 2, 3, 4, 5, 6, 7, 8}


def raise_status(status: int, what: str = "") -> None:
    if status == 0:
        return
    lib = _lib.load()
    code = _lib.error_code(status)
    msg = _lib.error_string(status)
    if status in _CONFIG_CODES:
        raise ConfigError(code, f"{msg}{(' ' + what) if what else ''}")
    if status == 9:
        raise TypeError(msg)
    if status == 13:
        raise RuntimeError(f"CUDA error {lib.btk_last_cuda_error()} in {what or 'btk'}")
    raise ValueError(f"{msg}{(' ' + what) if what else ''}")


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _DTYPES[t.dtype]
    except KeyError:
        raise TypeError(
            f"unsupported dtype {t.dtype}: the B200 kernels take float32, bfloat16, float16 or "
            "float64") from None


def to_device_tensor(scores, device=None) -> torch.Tensor:
    """Accept a torch tensor (any device) or array-like; return a CUDA tensor."""
    if isinstance(scores, torch.Tensor):
        t = scores
    else:
        t = torch.from_numpy(np.ascontiguousarray(host_array(scores)))
    if not t.is_cuda:
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        t = t.to(dev)
    return t


def host_array(scores) -> np.ndarray:
    """Array-like -> NumPy array.  NumPy float16/32/64 keep their dtype (each
    has an exact GPU path); Python lists / ints / other dtypes become float64,
    as the reference's _as_matrix does (exact.py:87-96)."""
    a = np.asarray(scores)
    if a.dtype not in (np.float16, np.float32, np.float64):
        a = a.astype(np.float64)
    return a


def as_rows(t: torch.Tensor, dim: int = -1):
    """(m, n) row view with unit inner stride, plus the leading shape.

    Mirrors reference exact.py:87-96: 1-D -> one row; empty rows rejected.
    """
    if t.ndim == 0:
        raise ValueError(f"scores must be a non-empty m x n matrix, got shape {tuple(t.shape)}")
    if t.ndim == 1:
        t = t.unsqueeze(0)
        lead = (1,)
    else:
        d = dim % t.ndim
        if d != t.ndim - 1:
            t = t.movedim(d, -1)
        lead = tuple(t.shape[:-1])
        t = t.reshape(-1, t.shape[-1])
    if t.shape[-1] == 0 or t.shape[0] == 0:
        raise ValueError(f"scores must be a non-empty m x n matrix, got shape {tuple(t.shape)}")
    if t.stride(-1) != 1 or (t.shape[0] > 1 and t.stride(0) < t.shape[1]):
        t = t.contiguous()
    esz = t.element_size()
    if t.data_ptr() % 16 or (t.stride(0) * esz) % 16:
        # keep the vector-load fast path available: 16-byte aligned rows
        t = t.contiguous() if (t.shape[1] * esz) % 16 == 0 else t
    return t, lead


def workspace(nbytes: int, device) -> torch.Tensor:
    """Device workspace (contents need not be initialised).  torch's
    caching allocator returns >= 512-byte aligned blocks."""
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


def stream_handle(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


_FLAGS = {}


def device_flag(device) -> torch.Tensor:
    """Non-finite flag per (device, current stream): int32, zero between
    calls (check_flag resets it when it reads a set bit).  Calls on one
    stream are ordered, and each reads its own launch's flag before the
    next call is issued, so the flag never carries a stale bit."""
    dev = torch.device(device)
    key = (dev, torch.cuda.current_stream(dev).cuda_stream)
    f = _FLAGS.get(key)
    if f is None:
        f = torch.zeros(1, dtype=torch.int32, device=dev)
        _FLAGS[key] = f
    return f


def check_flag(flag: torch.Tensor, reset: bool = False) -> None:
    v = int(flag.item())
    if v and reset:
        flag.zero_()
    if v & 1:
        raise NonFiniteInputError("scores contain NaN or infinity")
    if v & 2:
        raise ValueError("carried labels must lie in [0, 2**31 - 1] on the GPU path")
