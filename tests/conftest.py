import json
import os
import sys
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"

EPS = {"single": float(np.finfo(np.float32).eps), "double": float(np.finfo(np.float64).eps)}
DT = {"single": np.complex64, "double": np.complex128}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libtfft.so")


def gaussian(n, b, precision, seed):
    """tests/conftest.py:7-10 of the reference: re, im ~ N(0, 1) from default_rng(seed)."""
    rng = np.random.default_rng(seed)
    data = rng.standard_normal((b, n)) + 1j * rng.standard_normal((b, n))
    return data.astype(DT[precision])


def oracle_tol(precision, n, c=16.0):
    return c * EPS[precision] * np.log2(n)


def max_rel_error(got, ref):
    got = np.atleast_2d(got)
    ref = np.atleast_2d(ref)
    err = np.abs(got - ref).max(axis=1)
    scale = np.maximum(np.abs(ref).max(axis=1), 1e-300)
    return float((err / scale).max())


def rel_l2(got, ref):
    """north_star parity metric: relative L2 over the whole batch."""
    return float(np.linalg.norm((got - ref).ravel()) / max(np.linalg.norm(ref.ravel()), 1e-300))


def two_pass_group(precision, n):
    """Signals per ring group of the fused two-pass kernels (mirrors
    tfft_k3.cu k4_group): 16 MB of intermediate below 2^17, 32 MB from 2^17,
    with the per-size exceptions of the measured sweep."""
    bpc = 8 if precision == "single" else 16
    mb = 32 if n >= 2 ** 17 else 16
    if precision == "double" and n in (2 ** 17, 2 ** 18):
        mb = 20
    if precision == "double" and n == 2 ** 20:
        mb = 16
    if precision == "single" and n == 2 ** 20:
        mb = 24
    return max(1, (mb << 20) // (n * bpc))


def l2_tol(precision, n):
    """BASELINE.json north_star: 1e-5 log2N (FP32) / 1e-12 log2N (FP64)."""
    return (1e-5 if precision == "single" else 1e-12) * max(np.log2(n), 1.0)


@lru_cache(maxsize=1)
def golden():
    return json.loads((GOLDEN / "golden.json").read_text())


@lru_cache(maxsize=1)
def golden_fft_outputs():
    return dict(np.load(GOLDEN / "fft_outputs.npz"))


@lru_cache(maxsize=1)
def golden_abft_outputs():
    return dict(np.load(GOLDEN / "abft_outputs.npz"))


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device here (run with -m gpu on a B200)")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


# -- the reference conftest's helpers (reference tests/conftest.py), used by the
# vendored reference suite in tests/refsuite/ through ``from conftest import``


def gaussian_batch(n, b, precision, seed=0):
    from paper_2412_05824_b200 import SignalBatch
    return SignalBatch(gaussian(n, b, precision, seed))
