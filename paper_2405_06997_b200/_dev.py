"""Device-buffer plumbing: torch tensors are used only as CUDA allocations
(plus their stream); all computation happens in libwfpg_b200.so."""

import numpy as np

from . import _lib

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t

        if not t.cuda.is_available():
            raise _lib.WfpgError("a CUDA device is required (there is no CPU fallback)")
        _lib.load()
        _torch = t
    return _torch


def device():
    t = torch()
    return t.device("cuda", t.cuda.current_device())


_DT = {
    np.float64: "float64", np.int32: "int32", np.int64: "int64", np.uint8: "uint8",
    np.uint64: "uint64", np.uint32: "uint32", np.bool_: "bool",
}


def _tdtype(dtype):
    t = torch()
    return getattr(t, _DT[np.dtype(dtype).type])


def empty(shape, dtype):
    return torch().empty(shape, dtype=_tdtype(dtype), device=device())


def zeros(shape, dtype):
    return torch().zeros(shape, dtype=_tdtype(dtype), device=device())


def upload(a, dtype=None):
    a = np.ascontiguousarray(a, dtype=dtype)
    return torch().as_tensor(a, device=device())


def download(t):
    """Copy a device tensor to a numpy array (synchronising the stream)."""
    return t.detach().cpu().numpy()


def workspace(nbytes):
    return torch().empty(max(int(nbytes), 1), dtype=torch().uint8, device=device())


def stream():
    return _lib.stream_handle()


def sync():
    torch().cuda.current_stream().synchronize()
