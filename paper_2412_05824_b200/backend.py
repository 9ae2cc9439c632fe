"""Kernel backend registry (reference backend.py:1-66) with one entry: ``cuda``.

The reference registers a compiled Cython module and a numpy twin, each
exporting ``stockham_pass(src, dst, s, r, base, inverse)``
(_kernels.pyx:74-84). Here the only module is the sm_100a library: its
``stockham_pass`` runs one reference-order pass on the device (used by
``butterfly_radix`` and the boundary tests), while ``execute_plan`` and
``run_protected`` call the fused whole-plan kernels directly. There is no CPU
fallback; asking for any other backend raises ``RuntimeError`` exactly as the
reference does for an unavailable one (backend.py:30-37).
"""

from __future__ import annotations

import os
from contextlib import contextmanager

import numpy as np

from . import _device, _lib


class _CudaKernels:
    """Module-like object exposing the reference plugin signature."""

    COMPILED = True

    @staticmethod
    def stockham_pass(src, dst, s, r, base, inverse):
        """Apply one radix-r pass (r in {2, 4}) to every row of ``src``.

        ``src``/``dst``: 2-D C-contiguous arrays (numpy or CUDA tensors) of the
        same complex dtype; ``base``: omega_{s r}^q for q < s. Writes all of
        ``dst``; raises ValueError for other radices (_kernels.pyx:83-84).
        """
        if r not in (2, 4):
            raise ValueError(f"cuda kernel supports radix 2 and 4, got {r}")
        lib = _lib.load()
        t = _device.require_cuda()
        host_dst = None
        if _device.is_device_tensor(src):
            s_dev = src
            d_dev = dst
            b_dev = base if _device.is_device_tensor(base) else \
                t.as_tensor(np.ascontiguousarray(base), device="cuda").to(src.dtype)
        else:
            src = np.asarray(src)
            if src.ndim != 2 or not src.flags.c_contiguous or src.dtype not in (np.complex64, np.complex128):
                raise ValueError("src must be a 2-D C-contiguous complex64/complex128 array")
            if dst.shape != src.shape or dst.dtype != src.dtype:
                raise ValueError("dst must match src in shape and dtype")
            s_dev = _device.to_device(src)
            d_dev = t.empty_like(s_dev)
            b_dev = _device.to_device(np.ascontiguousarray(base, dtype=src.dtype))
            host_dst = dst
        prec = 0 if s_dev.dtype == t.complex64 else 1
        rows, n = int(s_dev.shape[0]), int(s_dev.shape[1])
        rc = lib.tfft_stockham_pass(s_dev.data_ptr(), d_dev.data_ptr(), rows, n, int(s), int(r), b_dev.data_ptr(),
                                    int(bool(inverse)), prec, _device.stream_handle())
        _lib.check(rc, "tfft_stockham_pass")
        if host_dst is not None:
            host_dst[...] = d_dev.cpu().numpy()


cuda = _CudaKernels()
_MODULES = {"cuda": cuda}


def available_backends():
    return tuple(sorted(_MODULES))


def _resolve(name):
    if name == "auto":
        return "cuda"
    if name not in _MODULES:
        raise RuntimeError(
            f"backend {name!r} is not available (have: {', '.join(available_backends())})"
        )
    return name


_active = _resolve(os.environ.get("RESILIENT_FFT_BACKEND", "auto"))


def active_backend() -> str:
    return _active


def kernel():
    """The module providing ``stockham_pass`` for the active backend."""
    return _MODULES[_active]


def set_backend(name: str) -> str:
    global _active
    previous = _active
    _active = _resolve(name)
    return previous


@contextmanager
def use_backend(name: str):
    previous = set_backend(name)
    try:
        yield
    finally:
        set_backend(previous)
