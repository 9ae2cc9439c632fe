"""Two-sided checksum protection over the B200 kernels (reference abft.py).

Same API and decisions as the reference: per-signal left checksums
(c_in = (e^T W) x vs c_out = e . y) detect and localise, location-weighted
right-side accumulators (s_in = sum w_j x_j, s_out = sum w_j y_j, w_j = global
index + 1) verify each window of ``group_size`` transactions and drive
delayed single-error correction, with recompute as the fallback.

Where the work happens:
  * the clean path is ONE fused kernel launch (tfft_protected): transform,
    per-signal c_in / c_out / floor / divergence, and each window's
    FFT(s_in)-vs-s_out group divergence, with no extra HBM sweeps
    (the reference re-reads X and Y with GEMVs, abft.py:648-665, 592-624);
  * when any signal triggers, the serial replay (abft.py:342-551) runs here on
    the host over O(B) scalars for the windows that hold a trigger, calling
    device primitives for every vector operation (weighted columns, the FP64
    correction FFT, the row patch + re-verify, group divergence, recompute).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

from . import _device, _lib
from . import fft_core
from .fft_core import (
    DTYPES,
    EPS,
    PRECISIONS,
    REAL_DTYPES,
    SignalBatch,
    Transaction,
    _check_plan_batch,
    _Counters,
    _output,
    device_execute,
    execute_plan,
    transaction_partition,
)

DEFAULT_DELTA = {"single": 1e-4, "double": 1e-10}
ORACLE_CAP = 4096
DIVERGENCE_FLOOR = 1e-30
LEFT_KINDS = ("wang", "jou", "ones")
MAX_SINGLE_WEIGHT = 2 ** 24


class Undecodable(ValueError):
    """Location decode failed: multi-error or noise-dominated divergence."""


def default_delta(precision: str) -> float:
    return DEFAULT_DELTA[precision]


@dataclass(frozen=True)
class EncodingVector:
    kind: str
    values: np.ndarray

    @property
    def length(self) -> int:
        return len(self.values)


def make_encoding_vector(kind, length, precision="double"):
    """abft.py:80-104 (host metadata; the kernels evaluate the same vectors).
    The vector is read-only, so equal requests share one object."""
    return _encoding_vector(kind, int(length), precision)


@lru_cache(maxsize=32)
def _encoding_vector(kind, length, precision):
    if length < 1:
        raise ValueError("length must be >= 1")
    if precision not in PRECISIONS:
        raise ValueError(f"unknown precision {precision!r}")
    dtype = DTYPES[precision]
    k = np.arange(length)
    if kind == "ones":
        values = np.ones(length, dtype=dtype)
    elif kind == "jou":
        values = np.exp((-2j * np.pi / length) * k).astype(dtype)
    elif kind == "wang":
        values = np.exp((-2j * np.pi / 3.0) * (k % 3)).astype(dtype)
    elif kind == "location":
        if precision == "single" and length > MAX_SINGLE_WEIGHT:
            raise ValueError("location vector longer than 2^24 is not exact in single precision")
        values = np.arange(1, length + 1, dtype=REAL_DTYPES[precision])
    else:
        raise ValueError(f"unknown encoding kind {kind!r}")
    values.setflags(write=False)
    return EncodingVector(kind, values)


@dataclass(frozen=True)
class LeftChecksumRow:
    kind: str
    n: int
    values: np.ndarray


def _standard_values(e):
    ref = make_encoding_vector(e.kind, e.length, "single" if e.values.dtype == np.complex64 else "double")
    return e.values.dtype == ref.values.dtype and np.array_equal(e.values, ref.values)


def precompute_left(e, n, precision=None, plan=None):
    """e^T W (abft.py:116-147).

    Named encodings use the closed form with integer phase reduction in
    extended precision (tfft_left_row); any other vector is transformed on the
    device in FP64 and rounded once.
    """
    if isinstance(e, str):
        if precision is None:
            raise ValueError("precision required when passing an encoding kind")
        e = make_encoding_vector(e, n, precision)
    if e.length != n:
        raise ValueError(f"encoding vector has length {e.length}, expected {n}")
    precision = "single" if e.values.dtype == np.complex64 else "double"
    dtype = DTYPES[precision]
    if e.kind in _lib.ENC and _standard_values(e):
        lib = _lib.load()
        row = np.empty(n, dtype=dtype)
        rc = lib.tfft_left_row(_lib.ENC[e.kind], n, 0 if precision == "single" else 1, row.ctypes.data)
        _lib.check(rc, "tfft_left_row")
    else:
        from .plan import build_plan, select_params

        p64 = build_plan(select_params(n, 1, "double"), "double")
        row = execute_plan(p64, SignalBatch(np.asarray(e.values, dtype=np.complex128)[None, :])).data[0]
        row = row.astype(dtype)
    row = np.ascontiguousarray(row)
    row.setflags(write=False)
    return LeftChecksumRow(e.kind, n, row)


@lru_cache(maxsize=8)
def _cached_left_row(kind, n, precision):
    return precompute_left(kind, n, precision)


def detect(reference, observed, delta, floor=DIVERGENCE_FLOOR):
    """abft.py:155-167."""
    if delta <= 0:
        raise ValueError("delta must be > 0")
    if not np.isfinite(observed):
        return True, float("inf")
    denom = max(abs(reference), floor, DIVERGENCE_FLOOR)
    divergence = float(abs(reference - observed) / denom)
    return divergence > delta, divergence


def locate(weighted, unweighted, batch=None, floor=DIVERGENCE_FLOOR):
    """abft.py:170-190: round(Re(weighted/unweighted)), the 1-based weight."""
    if not (np.isfinite(weighted) and np.isfinite(unweighted)):
        raise Undecodable("non-finite divergence")
    if abs(unweighted) <= floor:
        raise Undecodable("unweighted divergence is negligible")
    with np.errstate(over="ignore", invalid="ignore"):
        ratio = complex(weighted) / complex(unweighted)
    if not np.isfinite(ratio):
        raise Undecodable("divergence ratio is non-finite")
    if abs(ratio.imag) > 0.25:
        raise Undecodable(f"ratio {ratio:g} is not real")
    ident = int(round(float(ratio.real)))
    if batch is not None and not 1 <= ident <= batch:
        raise Undecodable(f"decoded id {ident} outside [1, {batch}]")
    return ident


@dataclass
class DetectionEvent:
    transaction: int
    signal: int
    divergence: float
    located: int | None = None


@dataclass
class RunStats:
    """Counters of abft.py:201-218; ``signal_sweeps`` counts logical sweeps."""

    signal_sweeps: int = 0
    verifications: int = 0
    corrections: int = 0
    recomputations: int = 0
    max_divergence: float = 0.0
    events: list = field(default_factory=list)

    def data_passes(self, b: int) -> float:
        return self.signal_sweeps / (2.0 * b)


@dataclass
class DetectionReport:
    triggered: bool
    divergence: float
    located: int | None
    corrected: bool
    uncorrectable: bool
    verification_index: int

    def __post_init__(self):
        if self.corrected and not self.triggered:
            raise ValueError("corrected implies triggered")
        if self.uncorrectable and (not self.triggered or self.corrected):
            raise ValueError("uncorrectable implies triggered and not corrected")


@dataclass
class _Pending:
    signal: int
    weight: float
    snap_in: object    # device column: this transaction's sum w_j x_j
    snap_out: object   # device column: this transaction's sum w_j y_j
    tx_index: int
    divergence: float
    located: int | None
    reference: complex
    floor: float


@dataclass
class ChecksumState:
    """Right-side accumulators and pending-error record (abft.py:250-261)."""

    group_size: int
    weights: np.ndarray
    s_in: object
    s_out: object
    residuals: dict = field(default_factory=dict)
    pending: _Pending | None = None
    transactions_seen: int = 0
    verifications: int = 0


# ---------------------------------------------------------------------------
# device helpers


def _prec(plan):
    return 0 if plan.precision == "single" else 1


class _DeviceSums:
    """Per-signal and per-window outputs of the fused kernel (tfft_sums), and
    the 4-word status block, carved from ONE device buffer laid out
    [counters 4 | win_div nwin | c_in 2b | c_out 2b | floors b | div b] so a
    clean run reads its status and window divergences in a single D2H copy."""

    def __init__(self, b, nwin):
        t = _device.require_cuda()
        nw = max(nwin, 1)
        self.nwin = nw
        self.buf = t.empty(4 + nw + 6 * b, dtype=t.float64, device="cuda")
        o = 4 + nw
        self.win_div = self.buf[4:o]
        self.c_in = self.buf[o:o + 2 * b]
        self.c_out = self.buf[o + 2 * b:o + 4 * b]
        self.floors = self.buf[o + 4 * b:o + 5 * b]
        self.div = self.buf[o + 5 * b:o + 6 * b]
        self.counters = fft_core._Counters(self.buf[:4].view(t.int64))

    def struct(self):
        return _lib.TfftSums(self.c_in.data_ptr(), self.c_out.data_ptr(), self.floors.data_ptr(),
                             self.div.data_ptr(), self.win_div.data_ptr())

    def status(self):
        """(counters dict, win_div) in one device-to-host copy."""
        h = self.buf[:4 + self.nwin].cpu().numpy()
        return fft_core._Counters.decode(h[:4].view(np.int64)), h[4:]

    def host(self):
        """(c_in, c_out, floors, div) on the host, in one device-to-host copy."""
        h = self.buf[4 + self.nwin:].cpu().numpy()
        b = h.size // 6
        return (h[:2 * b].view(np.complex128), h[2 * b:4 * b].view(np.complex128), h[4 * b:5 * b], h[5 * b:])


def _weighted_columns(plan, src, row0, row1, group, weight0=0):
    """(ngroups, n) device table of sum_{j in group} (weight0+j+1) src_j (abft.py:668-677)."""
    lib = _lib.load()
    t = _device.torch()
    ng = (row1 - row0 + group - 1) // group
    out = t.empty((max(ng, 1), plan.n), dtype=src.dtype, device=src.device)
    rc = lib.tfft_weighted_columns(_prec(plan), src.data_ptr(), plan.n, row0, row1, group, weight0, out.data_ptr(),
                                   _device.stream_handle())
    _lib.check(rc, "tfft_weighted_columns")
    return out


def _vec_add(plan, a, b):
    rc = _lib.load().tfft_vec_add(_prec(plan), a.data_ptr(), b.data_ptr(), plan.n, _device.stream_handle())
    _lib.check(rc, "tfft_vec_add")


def _jou_variant_dev(plan, x):
    y = _device.torch().empty_like(x)
    rc = _lib.load().tfft_jou_variant(plan.native, x.data_ptr(), y.data_ptr(), int(x.shape[0]),
                                      _device.stream_handle())
    _lib.check(rc, "tfft_jou_variant")
    return y


def _jou_undo_dev(plan, y):
    rc = _lib.load().tfft_jou_undo(plan.native, y.data_ptr(), int(y.shape[0]), _device.stream_handle())
    _lib.check(rc, "tfft_jou_undo")


def _correction(plan, pending, col, res):
    """abft.py:297-330 on the device: col = (snap_out - FFT64(snap_in)) / w_k;
    returns (usable, col) with the reference's usability rule."""
    lib = _lib.load()
    rc = lib.tfft_correction_column(plan.native, pending.snap_in.data_ptr(), pending.snap_out.data_ptr(),
                                    float(pending.weight), col.data_ptr(), res.data_ptr(), _device.stream_handle())
    _lib.check(rc, "tfft_correction_column")
    r = res.cpu().numpy()
    limit = 16.0 * np.log2(plan.n) * pending.floor * np.sqrt(plan.n)
    return bool(r[0] == 1.0) and float(r[1]) <= limit


def _patch(plan, y_row, col, enc_kind, res):
    """y_k -= col, then c_out = y_k . enc (abft.py:404-405)."""
    rc = _lib.load().tfft_patch_row(plan.native, y_row.data_ptr(), col.data_ptr(), _lib.ENC[enc_kind],
                                    res.data_ptr(), _device.stream_handle())
    _lib.check(rc, "tfft_patch_row")
    r = res.cpu().numpy()
    return complex(r[2], r[3])


def _group_div(plan, s_in, s_out, scratch, res):
    """FFT(s_in) in working precision vs s_out (abft.py:502-507)."""
    device_execute(plan, s_in.view(1, -1), scratch.view(1, -1))
    rc = _lib.load().tfft_group_divergence(_prec(plan), scratch.data_ptr(), s_out.data_ptr(), plan.n,
                                           res.data_ptr(), _device.stream_handle())
    _lib.check(rc, "tfft_group_divergence")
    return float(res[:1].cpu().numpy()[0])


class _ProtectedRun:
    """The serial decision replay of abft.py:342-551, vector state on the device."""

    def __init__(self, plan, source, out, delta, group_size, enc_kind, stats, sums_host, sig_off=0,
                 global_b=None):
        t = _device.torch()
        self.plan, self.source, self.out = plan, source, out
        self.delta, self.enc_kind, self.stats = delta, enc_kind, stats
        self.c_in, self.c_out, self.floors, self.div = sums_host
        b, n = int(source.shape[0]), plan.n
        # a batch shard keeps the GLOBAL location weights and indices
        self.sig_off = sig_off
        self.tx_off = sig_off // plan.bs
        self.global_b = global_b if global_b is not None else b
        self.state = ChecksumState(
            group_size=group_size,
            weights=np.arange(sig_off + 1, sig_off + b + 1, dtype=REAL_DTYPES[plan.precision]),
            s_in=t.zeros(n, dtype=source.dtype, device="cuda"),
            s_out=t.zeros(n, dtype=source.dtype, device="cuda"),
        )
        self.reports = []
        self.window_out_contribs = {}
        self.window_tx_count = 0
        self.window_corrected = False
        self.window_uncorrectable = False
        self._col = t.empty(n, dtype=source.dtype, device="cuda")
        self._ref = t.empty(n, dtype=source.dtype, device="cuda")
        self._res = _device.empty_f64(4)

    # -- correction machinery (abft.py:376-418) ------------------------------

    def _recompute_transaction(self, tx):
        rows = slice(tx.start, tx.stop)
        fft_core_run = _run_transaction_hook()
        fft_core_run(self.plan, self.source[rows], self.out[rows], "forward", None, tx.index, tx.start)
        self.stats.recomputations += 1
        self.stats.signal_sweeps += 2 * tx.size
        if tx.index in self.window_out_contribs:
            self.window_out_contribs[tx.index] = _weighted_columns(self.plan, self.out, tx.start, tx.stop,
                                                                   tx.size, self.sig_off)[0]
            acc = _device.torch().zeros_like(self.state.s_out)
            for v in self.window_out_contribs.values():
                _vec_add(self.plan, acc, v)
            self.state.s_out = acc

    def _apply_pending(self, tx_by_index, decontaminate):
        pending = self.state.pending
        self.state.pending = None
        k = pending.signal - self.sig_off
        col = self._col
        if _correction(self.plan, pending, col, self._res):
            observed = _patch(self.plan, self.out[k], col, self.enc_kind, self._res)
            still_bad, _ = detect(pending.reference, observed, self.delta, pending.floor)
            if not still_bad:
                self.stats.corrections += 1
                if decontaminate:
                    rc = _lib.load().tfft_vec_axpby(
                        _prec(self.plan), self.state.s_out.data_ptr(), self.plan.n, 1.0, 0.0,
                        self.state.s_out.data_ptr(), -float(pending.weight), 0.0, col.data_ptr(),
                        _device.stream_handle())
                    _lib.check(rc, "tfft_vec_axpby")
                self.window_corrected = True
                return True
        self._recompute_transaction(tx_by_index[pending.tx_index])
        self.window_uncorrectable = True
        return False

    # -- per-transaction replay (abft.py:422-489) -----------------------------

    def feed(self, tx, t_in, t_out, tx_by_index):
        state = self.state
        state.transactions_seen += 1
        self.window_tx_count += 1
        _vec_add(self.plan, state.s_in, t_in)
        _vec_add(self.plan, state.s_out, t_out)
        self.window_out_contribs[tx.index] = t_out
        hits = self.div[tx.start:tx.stop] > self.delta
        if hits.any():
            for gj in range(tx.start, tx.stop):
                state.residuals[gj] = complex(self.c_in[gj] - self.c_out[gj])
            triggered = [(tx.start + int(l), int(l), float(self.div[tx.start + int(l)]))
                         for l in np.nonzero(hits)[0]]
            self._handle_detections(tx, t_in, t_out, triggered, tx_by_index)
        if state.transactions_seen % state.group_size == 0:
            self._verify(tx_by_index)

    def batched_window(self, ntx, tx, k, div, decoded, group_div):
        """A window corrected by _batched_windows: the events, counters and
        report the serial replay produces for one trigger whose correction
        holds (abft.py:422-551: event, pending, patch + re-verify, decontaminated
        verification)."""
        self.state.transactions_seen += ntx
        event = DetectionEvent(tx.index + self.tx_off, k + self.sig_off, div, decoded)
        self.stats.events.append(event)
        self.stats.corrections += 1
        group_hit = group_div > self.delta
        divergence = max([div] + ([group_div] if group_hit else []))
        self.stats.verifications += 1
        self.state.verifications += 1
        self.reports.append(DetectionReport(triggered=True, divergence=float(divergence), located=k + self.sig_off,
                                            corrected=True, uncorrectable=False,
                                            verification_index=self.state.verifications - 1))

    def skip_clean_window(self, ntx, group_div):
        """A window without triggers: same report the replay would produce."""
        self.state.transactions_seen += ntx
        self._report_clean(group_div)

    def _report_clean(self, group_div):
        hit = group_div > self.delta
        self.stats.verifications += 1
        self.state.verifications += 1
        self.reports.append(DetectionReport(triggered=hit, divergence=float(group_div), located=None,
                                            corrected=False, uncorrectable=hit,
                                            verification_index=self.state.verifications - 1))

    def _handle_detections(self, tx, t_in, t_out, triggered, tx_by_index):
        res = self.state.residuals
        with np.errstate(over="ignore", invalid="ignore"):
            tx_res = sum(res[gj] for gj in range(tx.start, tx.stop))
            tx_wres = sum(float(self.state.weights[gj]) * res[gj] for gj in range(tx.start, tx.stop))
        try:
            decoded = locate(tx_wres, tx_res, batch=self.global_b) - 1
        except Undecodable:
            decoded = None
        if len(triggered) > 1:
            for gj, _, div in triggered:
                self.stats.events.append(DetectionEvent(tx.index + self.tx_off, gj + self.sig_off, div, None))
            if self.state.pending is not None:
                self._apply_pending(tx_by_index, decontaminate=True)
            self._recompute_transaction(tx)
            self.window_uncorrectable = True
            return
        gj, local, div = triggered[0]
        self.stats.events.append(DetectionEvent(tx.index + self.tx_off, gj + self.sig_off, div, decoded))
        if self.state.pending is not None:
            self._apply_pending(tx_by_index, decontaminate=False)
            self.state.s_in = t_in.clone()
            self.state.s_out = t_out.clone()
            self.window_out_contribs = {tx.index: t_out}
            self.window_tx_count = 1
        self.state.pending = _Pending(
            signal=gj + self.sig_off, weight=float(self.state.weights[gj]), snap_in=t_in, snap_out=t_out,
            tx_index=tx.index,
            divergence=div, located=gj + self.sig_off, reference=complex(self.c_in[gj]),
            floor=float(max(self.floors[gj], DIVERGENCE_FLOOR)))

    # -- verification boundaries (abft.py:493-551) ----------------------------

    def _verify(self, tx_by_index):
        state = self.state
        if self.window_tx_count == 0 and state.pending is None:
            return
        located = None
        if state.pending is not None:
            located = state.pending.located
            self._apply_pending(tx_by_index, decontaminate=True)
        group_div = _group_div(self.plan, state.s_in, state.s_out, self._ref, self._res)
        group_hit = group_div > self.delta
        events = [e for e in self.stats.events if e.signal - self.sig_off in state.residuals]
        if group_hit and not events and not self.window_corrected and not self.window_uncorrectable:
            self.window_uncorrectable = True
        divergence = max([e.divergence for e in events] + ([group_div] if group_hit else []), default=group_div)
        triggered = bool(events) or group_hit
        self.stats.verifications += 1
        state.verifications += 1
        self.reports.append(DetectionReport(
            triggered=triggered, divergence=float(divergence), located=located if triggered else None,
            corrected=self.window_corrected,
            uncorrectable=self.window_uncorrectable and not self.window_corrected,
            verification_index=state.verifications - 1))
        state.s_in.zero_()
        state.s_out.zero_()
        state.residuals.clear()
        self.window_out_contribs = {}
        self.window_tx_count = 0
        self.window_corrected = False
        self.window_uncorrectable = False

    def finish(self, tx_by_index):
        if self.state.transactions_seen % self.state.group_size != 0:
            self._verify(tx_by_index)
        elif self.state.pending is not None or self.window_tx_count:
            self._verify(tx_by_index)
        return self.reports


def _run_transaction_hook():
    # looked up at call time so tests can monkeypatch abft._run_transaction
    return globals()["_run_transaction"]


_run_transaction = fft_core._run_transaction


def correct_pending(state: ChecksumState, outputs: SignalBatch, plan, enc, delta, stats=None) -> DetectionReport:
    """Apply a held correction to ``outputs`` (abft.py:554-585)."""
    stats = stats if stats is not None else RunStats()
    if state.pending is None:
        return DetectionReport(triggered=False, divergence=0.0, located=None, corrected=False,
                               uncorrectable=False, verification_index=state.verifications)
    t = _device.torch()
    pending = state.pending
    for name in ("snap_in", "snap_out"):
        v = getattr(pending, name)
        if not _device.is_device_tensor(v):
            setattr(pending, name, _device.to_device(np.asarray(v, dtype=DTYPES[plan.precision])))
    col = t.empty(plan.n, dtype=pending.snap_in.dtype, device="cuda")
    res = _device.empty_f64(4)
    corrected = False
    y = _device.to_device(outputs.data)
    if _correction(plan, pending, col, res):
        observed = _patch(plan, y[pending.signal], col, enc.kind, res)
        still_bad, _ = detect(pending.reference, observed, delta, pending.floor)
        if still_bad:
            _vec_add(plan, y[pending.signal], col)
        else:
            corrected = True
            stats.corrections += 1
        if not outputs.on_device:
            outputs.data[pending.signal] = y[pending.signal].cpu().numpy()
    state.pending = None
    state.verifications += 1
    return DetectionReport(triggered=True, divergence=pending.divergence, located=pending.located,
                           corrected=corrected, uncorrectable=not corrected,
                           verification_index=state.verifications - 1)


# test hook: force the per-transaction replay engine even on clean runs
_FORCE_ENGINE = False


def _prepare(plan, batch, e_left, delta, sig_off=0, global_b=None):
    """abft.py:627-645 (the non-finite check happens in-kernel). A shard of a
    larger batch checks the single-precision weight limit on the GLOBAL
    signal indices (its weights are sig_off + j + 1)."""
    _check_plan_batch(plan, batch, "forward")
    precision = batch.precision
    if delta is None:
        delta = default_delta(precision)
    kind = e_left.kind if isinstance(e_left, EncodingVector) else e_left
    if kind not in LEFT_KINDS:
        raise ValueError(f"left encoding must be one of {LEFT_KINDS}, got {kind!r}")
    top = max(sig_off + batch.b, global_b if global_b is not None else 0)
    if precision == "single" and top > MAX_SINGLE_WEIGHT:
        raise ValueError("location weights above 2^24 are not exact in single precision")
    enc = e_left if isinstance(e_left, EncodingVector) else make_encoding_vector(kind, batch.n, precision)
    return precision, delta, kind, enc


def _fault_args(faults):
    return fft_core._fault_array(faults), len(faults)


def protected_device(plan, src, y, *, kind="wang", delta, group_size, faults=(), signal_offset=0,
                     counters=None, sums=None, stream=None):
    """One tfft_protected launch on device tensors (no synchronisation)."""
    lib = _lib.load()
    fa, nf = _fault_args(list(faults))
    rc = lib.tfft_protected(plan.native, src.data_ptr(), y.data_ptr(), int(src.shape[0]), int(signal_offset),
                            _lib.ENC[kind], float(delta), int(group_size), fa, nf, ctypes.byref(sums.struct()),
                            counters.ptr, stream if stream is not None else _device.stream_handle())
    _lib.check(rc, "tfft_protected")


def run_protected(plan, batch, e_left="wang", delta=None, group_size=1, mode="fused", *, workers=1,
                  injector=None, stats=None, out=None):
    """Transform under two-sided checksum protection (abft.py:690-752).

    Fault-free runs return outputs bitwise equal to ``execute_plan`` (the
    fused kernel runs the identical butterfly code) and untriggered reports.
    """
    return _protected(plan, batch, e_left, delta, group_size, mode, injector, stats, out, 0, None)


def _protected(plan, batch, e_left, delta, group_size, mode, injector, stats, out, sig_off, global_b):
    """run_protected over a (possibly sharded) batch: rows are global signals
    [sig_off, sig_off + b) of a global batch of ``global_b`` signals."""
    if group_size < 1:
        raise ValueError("group size must be >= 1")
    if mode not in ("fused", "per-transaction"):
        raise ValueError(f"unknown mode {mode!r}")
    precision, delta, kind, enc = _prepare(plan, batch, e_left, delta, sig_off, global_b)
    stats = stats if stats is not None else RunStats()
    t = _device.require_cuda()
    x = _device.to_device(batch.data)
    source = _jou_variant_dev(plan, x) if kind == "jou" else x
    y = t.empty_like(x)
    ntx = (batch.b + plan.bs - 1) // plan.bs  # the Transaction objects only when the replay runs
    nwin = (ntx + group_size - 1) // group_size
    sums = _DeviceSums(batch.b, nwin)
    tx_off = sig_off // plan.bs
    faults = injector._collect(tx_off, tx_off + ntx) if injector is not None else []
    protected_device(plan, source, y, kind=kind, delta=delta, group_size=group_size, faults=faults,
                     counters=sums.counters, sums=sums, signal_offset=sig_off)
    c, win_div = sums.status()
    if c["nonfinite"]:
        for f in faults:
            f.fired = False
        raise ValueError("batch contains non-finite values")
    stats.signal_sweeps += 2 * batch.b
    if mode == "per-transaction":
        stats.signal_sweeps += 2 * batch.b  # unfused checksum reductions
    stats.max_divergence = max(stats.max_divergence, c["max_div"])

    if c["triggered"] == 0 and not _FORCE_ENGINE:
        reports = []
        for w in range(nwin):
            g = float(win_div[w])
            stats.verifications += 1
            reports.append(DetectionReport(triggered=g > delta, divergence=g, located=None, corrected=False,
                                           uncorrectable=g > delta, verification_index=w))
    else:
        host = sums.host()
        run = _ProtectedRun(plan, source, y, delta, group_size, kind, stats, host, sig_off, global_b)
        txs = _TxTable(plan.bs, batch.b)
        tx_by_index = txs
        div = host[3]
        batched = _batched_windows(plan, source, y, batch, txs, ntx, nwin, group_size, div, host, kind, delta,
                                   sig_off, run)
        win_hit = np.zeros(nwin, dtype=bool)
        win_hit[(np.flatnonzero(div > delta) // plan.bs) // group_size] = True
        with np.errstate(over="ignore", invalid="ignore"):
            for w in range(nwin):
                first, last = w * group_size, min((w + 1) * group_size, ntx)
                if not _FORCE_ENGINE and not win_hit[w]:
                    run.skip_clean_window(last - first, float(win_div[w]))
                    continue
                a, b = txs[first].start, txs[last - 1].stop
                if w in batched:
                    run.batched_window(last - first, *batched[w])
                    continue
                t_in = _weighted_columns(plan, source, a, b, plan.bs, sig_off)
                t_out = _weighted_columns(plan, y, a, b, plan.bs, sig_off)
                for i, ti in enumerate(range(first, last)):
                    run.feed(txs[ti], t_in[i], t_out[i], tx_by_index)
            reports = run.finish(tx_by_index)
    if kind == "jou":
        _jou_undo_dev(plan, y)
    return _output(batch, y, out), reports


class _TxTable:
    """transaction_partition's entries made on demand (fft_core.py:245-252):
    a triggered run touches a few of the ntx transactions, and building all
    of them costs ~1 us each on the host."""

    def __init__(self, bs, b):
        self.bs, self.b = bs, b

    def __getitem__(self, i):
        start = i * self.bs
        return Transaction(i, start, min(start + self.bs, self.b))


def _batched_windows(plan, source, y, batch, txs, ntx, nwin, T, div, host, kind, delta, sig_off, run):
    """The replay's common case for all windows at once (tfft_correct_windows):
    windows whose only trigger is one signal are corrected in one batched
    call -- snapshot sums, FP64 correction FFTs, usability, patch, re-verify,
    decontaminated window check -- instead of per-event host round trips.
    Returns {window: (tx, signal, divergence, decoded, group_div)} for the
    windows it corrected; every other triggered window (several triggers,
    an unusable column, a failed re-verify) goes through the serial replay,
    with y untouched by this call, so decisions stay the reference's."""
    if _FORCE_ENGINE or kind not in ("wang", "ones") or os.environ.get("TFFT_NO_BATCHED_CORRECTION"):
        return {}
    hits = np.flatnonzero(div > delta)
    if hits.size == 0:
        return {}
    bs = plan.bs
    win_of = (hits // bs) // T
    wins, first_idx, counts = np.unique(win_of, return_index=True, return_counts=True)
    sel = counts == 1
    if not sel.any():
        return {}
    wsel = wins[sel]
    k = hits[first_idx[sel]]
    c_in, c_out, floors = host[0], host[1], host[2]
    b = batch.b
    r0 = (k // bs) * bs
    r1 = np.minimum(r0 + bs, b)
    w0 = wsel * T * bs
    w1 = np.minimum((wsel + 1) * T * bs, b)
    desc = np.ascontiguousarray(np.stack([k, r0, r1, wsel, w0, w1], axis=1).astype(np.int64))
    weights = np.asarray(run.state.weights)
    par = np.ascontiguousarray(np.stack([weights[k].astype(np.float64), np.maximum(floors[k], DIVERGENCE_FLOOR),
                                         c_in[k].real, c_in[k].imag], axis=1).astype(np.float64))
    count = int(k.size)
    out = np.zeros(4 * count, dtype=np.float64)
    lib = _lib.load()
    rc = lib.tfft_correct_windows(plan.native, source.data_ptr(), y.data_ptr(), int(sig_off), count,
                                  desc.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                  par.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _lib.ENC[kind], float(delta),
                                  out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _device.stream_handle())
    _lib.check(rc, "tfft_correct_windows")
    meta = [(int(wsel[i]), txs[int(k[i]) // bs], int(k[i])) for i in range(count)]
    res = {}
    ok = out.reshape(count, 4)
    done = [int(i) for i in np.flatnonzero(ok[:, 0] == 1.0)]  # others: the serial replay handles the window
    if not done:
        return res
    # the transaction residual sums of _handle_detections (abft.py:463-466),
    # same sequential order, vectorised across the windows
    weights = np.asarray(run.state.weights, dtype=np.float64)
    starts = np.array([meta[i][1].start for i in done])
    sizes = np.array([meta[i][1].stop - meta[i][1].start for i in done])
    with np.errstate(over="ignore", invalid="ignore"):
        cols = np.arange(int(sizes.max()))
        live = cols[None, :] < sizes[:, None]
        idx = np.where(live, starts[:, None] + cols[None, :], starts[:, None])
        r = np.where(live, c_in[idx] - c_out[idx], 0)
        # cumulative sums run left to right: the sequential order of sum()
        tx_res = np.cumsum(r, axis=1)[:, -1]
        tx_wres = np.cumsum(np.where(live, weights[idx], 0.0) * r, axis=1)[:, -1]
        for q, i in enumerate(done):
            w, tx, k = meta[i]
            try:
                decoded = locate(complex(tx_wres[q]), complex(tx_res[q]), batch=run.global_b) - 1
            except Undecodable:
                decoded = None
            res[w] = (tx, k, float(div[k]), decoded, float(ok[i, 2]))
    return res


def run_offline(plan, batch, e_left="wang", delta=None, *, workers=1, injector=None, stats=None, out=None):
    """One-sided baseline (abft.py:755-838): transform, then separate checksum
    sweeps over X and Y, recompute-on-detect with a 3-attempt abort."""
    precision, delta, kind, enc = _prepare(plan, batch, e_left, delta)
    stats = stats if stats is not None else RunStats()
    t = _device.require_cuda()
    lib = _lib.load()
    x = _device.to_device(batch.data)
    source = _jou_variant_dev(plan, x) if kind == "jou" else x
    y = t.empty_like(x)
    txs = transaction_partition(plan, batch)
    faults = injector._collect(0, len(txs)) if injector is not None else []
    counters = _Counters()
    device_execute(plan, source, y, faults=faults, counters=counters)
    if counters.read()["nonfinite"]:
        for f in faults:
            f.fired = False
        raise ValueError("batch contains non-finite values")
    stats.signal_sweeps += 2 * batch.b
    sums = _DeviceSums(batch.b, 1)
    st = sums.struct()

    def checksums(row0, nrows):
        rc = lib.tfft_row_checksums(plan.native, source.data_ptr(), y.data_ptr(), row0, nrows, _lib.ENC[kind],
                                    float(delta), ctypes.byref(st), None, 0, _device.stream_handle())
        _lib.check(rc, "tfft_row_checksums")

    checksums(0, batch.b)  # the post-hoc input + output passes
    c_in, c_out, floors, _ = sums.host()
    reports = []
    for tx in txs:
        stats.signal_sweeps += 2 * tx.size
        triggered = []
        for local, gj in enumerate(range(tx.start, tx.stop)):
            hit, div = detect(c_in[gj], c_out[gj], delta, max(floors[gj], DIVERGENCE_FLOOR))
            stats.max_divergence = max(stats.max_divergence, div)
            if hit:
                triggered.append((gj, local, div))
                stats.events.append(DetectionEvent(tx.index, gj, div, gj))
        for gj, local, div in triggered:
            for attempt in range(3):
                _run_transaction_hook()(plan, source[gj:gj + 1], y[gj:gj + 1], "forward", None, tx.index, gj)
                stats.recomputations += 1
                stats.signal_sweeps += 2
                checksums(gj, 1)
                observed = complex(*sums.c_out[2 * gj:2 * gj + 2].cpu().numpy())
                still_bad, _ = detect(c_in[gj], observed, delta, max(floors[gj], DIVERGENCE_FLOOR))
                if not still_bad:
                    break
            else:
                raise RuntimeError(
                    f"signal {gj} still diverges after 3 recomputations; suspecting a persistent fault, aborting")
        stats.verifications += 1
        reports.append(DetectionReport(triggered=bool(triggered),
                                       divergence=max((d for _, _, d in triggered), default=0.0),
                                       located=triggered[0][0] if triggered else None,
                                       corrected=bool(triggered), uncorrectable=False,
                                       verification_index=tx.index))
    if kind == "jou":
        _jou_undo_dev(plan, y)
    return _output(batch, y, out), reports
