"""ctypes binding of libtfft.so (the C ABI declared in include/tfft.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every transform raises ``RuntimeError`` (the reference backend
registry raises the same way for an unavailable backend, backend.py:30-37).
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libtfft.so"

OK, EINVAL, ENONFINITE, ECUDA, ENOMEM, EUNSUPPORTED = range(6)
SINGLE, DOUBLE = 0, 1
ENC = {"wang": 0, "ones": 1, "jou": 2}

c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int32
c_int = ctypes.c_int
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
c_u64p = ctypes.POINTER(ctypes.c_uint64)


class TfftFault(ctypes.Structure):
    _fields_ = [("transaction", c_i64), ("signal", c_i64), ("element", c_i64),
                ("stage", c_i32), ("part", c_i32), ("bit", c_i32), ("reserved", c_i32)]


class TfftSums(ctypes.Structure):
    _fields_ = [("c_in", c_vp), ("c_out", c_vp), ("floors", c_vp), ("div", c_vp), ("win_div", c_vp)]


# symbol -> (restype, argtypes); every symbol include/tfft.h declares
SIGNATURES = {
    "tfft_version": (c_int, []),
    "tfft_last_error": (ctypes.c_char_p, []),
    "tfft_launch_count": (ctypes.c_uint64, []),
    "tfft_plan_create": (c_int, [c_i64, c_int, c_int, ctypes.POINTER(c_i64), ctypes.POINTER(c_i32), c_i64,
                                 ctypes.POINTER(c_vp)]),
    "tfft_plan_destroy": (c_int, [c_vp]),
    "tfft_debug_skew_twiddle": (c_int, [c_vp]),
    "tfft_execute": (c_int, [c_vp, c_vp, c_vp, c_i64, c_int, c_i64, ctypes.POINTER(TfftFault), c_int, c_vp, c_vp]),
    "tfft_protected": (c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_int, c_dbl, c_i64, ctypes.POINTER(TfftFault),
                               c_int, ctypes.POINTER(TfftSums), c_vp, c_vp]),
    "tfft_stockham_pass": (c_int, [c_vp, c_vp, c_i64, c_i64, c_i64, c_int, c_vp, c_int, c_int, c_vp]),
    "tfft_left_row": (c_int, [c_int, c_i64, c_int, c_vp]),
    "tfft_weighted_columns": (c_int, [c_int, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp]),
    "tfft_vec_add": (c_int, [c_int, c_vp, c_vp, c_i64, c_vp]),
    "tfft_vec_axpby": (c_int, [c_int, c_vp, c_i64, c_dbl, c_dbl, c_vp, c_dbl, c_dbl, c_vp, c_vp]),
    "tfft_group_divergence": (c_int, [c_int, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "tfft_correction_column": (c_int, [c_vp, c_vp, c_vp, c_dbl, c_vp, c_vp, c_vp]),
    "tfft_patch_row": (c_int, [c_vp, c_vp, c_vp, c_int, c_vp, c_vp]),
    "tfft_correct_windows": (c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, ctypes.POINTER(c_i64), ctypes.POINTER(c_dbl),
                                     c_int, c_dbl, ctypes.POINTER(c_dbl), c_vp]),
    "tfft_row_checksums": (c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_int, c_dbl, ctypes.POINTER(TfftSums), c_vp,
                                   c_int, c_vp]),
    "tfft_jou_variant": (c_int, [c_vp, c_vp, c_vp, c_i64, c_vp]),
    "tfft_jou_undo": (c_int, [c_vp, c_vp, c_i64, c_vp]),
    "tfft_allreduce_stats": (c_int, [c_vp, c_int, c_vp, c_vp, c_vp]),
}

_lib = None
_lock = threading.Lock()


class TfftError(RuntimeError):
    pass


def load(path=None):
    """Load (once) and type the library; raises RuntimeError when absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        # TFFT_LIB: an alternative build of the same C ABI (timing experiments, tools/)
        p = Path(path) if path else Path(os.environ.get("TFFT_LIB") or LIB_PATH)
        if not p.exists():
            raise RuntimeError(
                f"libtfft.so not found at {p}; build it with `python -c \"import __graft_entry__ as g; g.build()\"`"
            )
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc, what=""):
    """Map a C status to the reference's exception types."""
    if rc == OK:
        return
    msg = _lib.tfft_last_error().decode(errors="replace") if _lib is not None else ""
    text = f"{what}: {msg}" if what else msg
    if rc in (EINVAL, ENONFINITE, EUNSUPPORTED):
        raise ValueError(text)
    raise TfftError(text)
