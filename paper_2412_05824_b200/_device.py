"""Device plumbing: torch supplies CUDA memory and streams, nothing else.

Signal data crosses the host/device boundary here (numpy <-> torch CUDA
tensors); every transform and checksum runs in libtfft.so.
"""

from __future__ import annotations

import numpy as np

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 kernels have no CPU fallback")
    return t


TORCH_DTYPES = {}


def torch_dtype(np_dtype):
    t = torch()
    return {np.dtype(np.complex64): t.complex64, np.dtype(np.complex128): t.complex128}[np.dtype(np_dtype)]


def numpy_dtype(torch_dt):
    t = torch()
    return {t.complex64: np.complex64, t.complex128: np.complex128}[torch_dt]


def is_device_tensor(a):
    if _torch is None:
        try:
            import torch as t  # noqa: F401
        except ImportError:
            return False
    t = torch()
    return isinstance(a, t.Tensor) and a.is_cuda


def to_device(a):
    """numpy (or host tensor) -> contiguous CUDA tensor; CUDA tensors pass through."""
    t = require_cuda()
    if isinstance(a, t.Tensor):
        return a.contiguous() if a.is_cuda else a.to("cuda").contiguous()
    arr = np.ascontiguousarray(a)
    host = t.from_numpy(arr)
    return host.to("cuda", non_blocking=False)


def to_host(dev, out=None):
    """CUDA tensor -> numpy (synchronous)."""
    a = dev.cpu().numpy() if out is None else out
    if out is not None:
        out[...] = dev.cpu().numpy()
    return a


def ptr(tensor):
    return None if tensor is None else tensor.data_ptr()


def stream_handle():
    t = torch()
    return t.cuda.current_stream().cuda_stream


def empty(shape, np_dtype):
    t = require_cuda()
    return t.empty(shape, dtype=torch_dtype(np_dtype) if not isinstance(np_dtype, t.dtype) else np_dtype,
                   device="cuda")


def empty_f64(shape):
    t = require_cuda()
    return t.empty(shape, dtype=t.float64, device="cuda")


def zeros_u64(n):
    t = require_cuda()
    return t.zeros(n, dtype=t.int64, device="cuda")
