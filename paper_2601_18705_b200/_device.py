"""Device plumbing: which CUDA device, the current stream, fp64 tensors.

The B200 path is CUDA-only: ``device()`` raises when no GPU is visible
instead of silently computing on the host.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib

_DEV = None


def device():
    global _DEV
    if _DEV is None:
        if not torch.cuda.is_available():
            raise RuntimeError("the B200 DLR-SN path needs a CUDA device (no CPU fallback)")
        _DEV = torch.device("cuda", torch.cuda.current_device())
        _lib.load()
    return _DEV


def set_device(index):
    global _DEV
    torch.cuda.set_device(index)
    _DEV = torch.device("cuda", index)
    _lib.load()


def stream():
    """Raw handle of the current CUDA stream (the C-ABI's dlrsn_stream_t)."""
    return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(device().index))


def as_device(x, n=None, dtype=torch.float64):
    """fp64 contiguous CUDA tensor from numpy / torch / scalar (scalars
    broadcast to length ``n``)."""
    if isinstance(x, torch.Tensor):
        if x.dtype == dtype and x.is_cuda and x.ndim > 0 and x.is_contiguous():
            return x  # fast path: already a device tensor of the right kind
        t = x.to(device=device(), dtype=dtype)
    else:
        a = np.asarray(x, dtype=np.float64 if dtype == torch.float64 else None)
        if a.ndim == 0 and n is not None:
            a = np.full(n, float(a))
        t = torch.from_numpy(np.array(a, copy=True, order="C")).to(device=device(), dtype=dtype)
    if t.ndim == 0 and n is not None:
        t = t.expand(n)
    return t.contiguous()


def upload(a, dtype=None):
    """Host array -> device without a stream sync: stage through pinned
    memory and copy asynchronously (torch keeps the pinned block alive until
    the copy has executed).  A pageable H2D copy would wait for the stream."""
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.pin_memory().to(device(), non_blocking=True)


_CONST = {}


def cached_upload(key, make):
    """Device copy of a constant host array, uploaded once per device."""
    k = (torch.cuda.current_device(), key)
    t = _CONST.get(k)
    if t is None:
        t = upload(make())
        _CONST[k] = t
    return t


def zeros(*shape, dtype=torch.float64):
    return torch.zeros(*shape, dtype=dtype, device=device())


def empty(*shape, dtype=torch.float64):
    return torch.empty(*shape, dtype=dtype, device=device())


def to_numpy(t):
    if isinstance(t, torch.Tensor):
        return t.detach().cpu().numpy()
    return np.asarray(t)
