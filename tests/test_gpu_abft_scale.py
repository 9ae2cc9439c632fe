"""GPU: the fused / one-sweep ABFT paths at batch sizes where the work split
matters (K5 windows split into many pieces finished by the last-arriving
piece; K4 sizes through the one-sweep checksum kernel). Checked against FP64
numpy recomputations of the reference's quantities (abft.py:592-665) and
against the detection/correction contract: fault-free runs are bitwise equal
to execute_plan with no trigger, a single injected flip is detected at its
(transaction, signal) and corrected."""

import numpy as np
import pytest

from conftest import gaussian, max_rel_error, oracle_tol

pytestmark = pytest.mark.gpu


def _tf():
    import paper_2412_05824_b200 as tf
    return tf


CASES = [
    # precision, n, b, T   (K5 multi-piece windows; K4 + one-sweep sums)
    ("single", 1024, 8192, 64),
    ("single", 4096, 2048, 8),
    ("double", 2048, 2048, 16),
    ("single", 65536, 96, 4),
    ("double", 16384, 128, 4),
]


def _left_row(n, dtype):
    """e^T W for the wang encoding, FP64 (abft.py:80-152): row[k] = sum_j e_j w_N^{jk}."""
    j = np.arange(n)
    e = np.exp(-2j * np.pi * (j % 3) / 3)
    return np.fft.fft(e).astype(np.complex128)  # sum_j e_j exp(-2 pi i j k / n)


def _route(mode, n, monkeypatch):
    """default; the fused K5 or the one-sweep route for single-pass sizes; the
    opt-in fused K4 C tiles (TFFT_K4_ABFT=1) for two-pass sizes"""
    if mode == "k4fused":
        if n <= 4096:
            pytest.skip("two-pass sizes only")
        monkeypatch.setenv("TFFT_K4_ABFT", "1")
    elif mode != "default":
        if n > 4096:
            pytest.skip("no fused kernel at this size")
        # both protected routes for the fused sizes (tfft_api.cu abft_use_sweep)
        monkeypatch.setenv("TFFT_ABFT_SWEEP", "1" if mode == "sweep" else "0")


@pytest.mark.parametrize("mode", ["default", "fused", "sweep", "k4fused"])
@pytest.mark.parametrize("precision,n,b,T", CASES, ids=lambda v: str(v))
def test_protected_sums_match_fp64_recomputation(precision, n, b, T, mode, monkeypatch):
    import torch

    _route(mode, n, monkeypatch)
    tf = _tf()
    from paper_2412_05824_b200 import abft as A, fft_core
    x = gaussian(n, b, precision, seed=n + b)
    plan = tf.build_plan(tf.select_params(n, b, precision), precision)
    dt = torch.complex64 if precision == "single" else torch.complex128
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    yp = torch.empty_like(xd)
    bs = plan.bs
    W = T * bs
    nwin = -(-b // W)
    sums = A._DeviceSums(b, nwin)
    ctr = fft_core._Counters()
    A.protected_device(plan, xd, yd, delta=A.default_delta(precision), group_size=T, counters=ctr, sums=sums)
    fft_core.device_execute(plan, xd, yp)
    torch.cuda.synchronize()
    assert torch.equal(yd, yp), "fault-free protected output must equal the plain transform bitwise"
    y = yd.cpu().numpy().astype(np.complex128)
    x64 = x.astype(np.complex128)
    # per-signal two-sided checksums
    row = _left_row(n, dt)
    enc = np.exp(-2j * np.pi * (np.arange(n) % 3) / 3)
    c_in = x64 @ row
    c_out = y @ enc
    got_in = sums.c_in.cpu().numpy().view(np.complex128)
    got_out = sums.c_out.cpu().numpy().view(np.complex128)
    scale = np.linalg.norm(x64, axis=1) * np.sqrt(n)
    tol = 64 * oracle_tol(precision, n)
    assert np.all(np.abs(got_in - c_in) <= tol * scale)
    assert np.all(np.abs(got_out - c_out) <= tol * scale)
    floors = np.linalg.norm(x64, axis=1) / np.sqrt(n)
    assert np.allclose(sums.floors.cpu().numpy(), floors, rtol=1e-4 if precision == "single" else 1e-10)
    div = sums.div.cpu().numpy()
    assert np.all(np.isfinite(div)) and div.max() < A.default_delta(precision)
    # per-window group divergence: ||FFT(s_in) - s_out|| / ||FFT(s_in)|| with w_j = j + 1
    w = np.arange(1, b + 1, dtype=np.float64)
    wd = sums.win_div.cpu().numpy()
    for k in range(nwin):
        sl = slice(k * W, min((k + 1) * W, b))
        s_in = (w[sl, None] * x64[sl]).sum(0)
        s_out = (w[sl, None] * y[sl]).sum(0)
        ref = np.fft.fft(s_in)
        want = np.linalg.norm(ref - s_out) / np.linalg.norm(ref)
        assert np.isfinite(wd[k]) and wd[k] < A.default_delta(precision)
        assert abs(wd[k] - want) <= 16 * oracle_tol(precision, n) + 4 * want
    assert ctr.read()["triggered"] == 0  # nothing triggered


@pytest.mark.parametrize("mode", ["default", "fused", "sweep", "k4fused"])
@pytest.mark.parametrize("precision,n,b,T", CASES, ids=lambda v: str(v))
def test_single_fault_detected_and_corrected_at_scale(precision, n, b, T, mode, monkeypatch):
    _route(mode, n, monkeypatch)
    tf = _tf()
    x = gaussian(n, b, precision, seed=3 * n + b)
    plan = tf.build_plan(tf.select_params(n, b, precision), precision)
    batch = tf.SignalBatch(x)
    clean = tf.execute_plan(plan, batch).data
    sig = (b * 5) // 7
    tx = sig // plan.bs
    # an exponent bit that is 0 in the row's largest element: the flip scales
    # it up by 2^8..2^16 (finite), far above delta for any left-row weight (a
    # small flip can legitimately stay below delta -- the reference then only
    # triggers the window, not the signal)
    el = int(np.argmax(np.abs(x[sig].real)))
    if precision == "single":
        u = int(np.array([x[sig, el].real], dtype=np.float32).view(np.uint32)[0])
        bit = next(k for k in (26, 27, 25) if not (u >> k) & 1)
    else:
        u = int(np.array([x[sig, el].real], dtype=np.float64).view(np.uint64)[0])
        bit = next(k for k in (55, 56, 54) if not (u >> k) & 1)
    spec = tf.FaultSpec(transaction=tx, signal=sig, element=el, stage=0, part="re", bit=bit)
    inj = tf.FaultInjector()
    inj.arm(spec, plan=plan, batch=batch)
    stats = tf.RunStats()
    out, reports = tf.run_protected(plan, batch, group_size=T, injector=inj, stats=stats)
    assert [(e.transaction, e.signal) for e in stats.events] == [(tx, sig)]
    assert stats.corrections + stats.recomputations == 1
    trig = [i for i, r in enumerate(reports) if r.triggered]
    assert trig == [tx // T]
    assert max_rel_error(out.data, clean) <= 2 * oracle_tol(precision, n)
