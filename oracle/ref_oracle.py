"""TEST INFRASTRUCTURE ONLY — CPU oracle for the batched FFT ± two-sided ABFT path.

This module restates, in numpy, the reference package ``resilient-fft`` 0.1.0
(`/root/reference/pkg/src/resilient_fft`) for the north-star path: plan
selection, the radix-4/2 Stockham sweep, stage-boundary fault strikes, the
two-sided checksum protection with its serial replay engine, and the offline
one-sided baseline. It is the CHECKER: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it. The product package
(``paper_2412_05824_b200``) never imports anything under ``oracle/``.

Parity pin: ``tests/test_oracle_golden.py`` checks this restatement against
``tests/golden/`` (fixtures produced by calling the reference's own API, see
``tests/golden/make_golden.py``): transform outputs, strike layouts, and the
exact event / counter / report sets of 48 scripted and 400 seeded protected
runs.

When ``oracle/_ref/`` holds the reference's own compiled pass kernel (built by
``oracle/build_ref.sh`` from the reference's ``_kernels.pyx``), ``use_ref_kernel``
switches the per-pass arithmetic to it; that is the "reference" CPU baseline.
"""

from __future__ import annotations

import functools
import glob
import importlib.util
import math
import os
from dataclasses import dataclass, field

import numpy as np

DTYPES = {"single": np.complex64, "double": np.complex128}
RDTYPES = {"single": np.float32, "double": np.float64}
EPS = {"single": float(np.finfo(np.float32).eps), "double": float(np.finfo(np.float64).eps)}
DEFAULT_DELTA = {"single": 1e-4, "double": 1e-10}   # abft.py:41
FLOOR = 1e-30                                         # abft.py:48
ORACLE_CAP = 4096                                     # abft.py:45
MAX_SINGLE_WEIGHT = 2 ** 24                           # abft.py:59

# plan_table.txt:7-9 (curated rows = Table 1 of the paper)
CURATED = {
    1024: ((1024,), (8,), 1),
    131072: ((256, 512), (16, 16), 8),
    8388608: ((256, 128, 256), (16, 16, 16), 16),
}


def precision_of(a):
    return "single" if a.dtype == np.complex64 else "double"


# ---------------------------------------------------------------------------
# plan selection — plan.py:109-145


def stage_exponents(log2n):
    """plan.py:109-118: one stage to 2^13, two to 2^22, three beyond."""
    if log2n <= 13:
        return (log2n,)
    if log2n <= 22:
        a = (log2n + 1) // 2
        return (a, log2n - a)
    a = (log2n + 2) // 3
    rest = log2n - a
    b = (rest + 1) // 2
    return tuple(sorted((a, b, rest - b), reverse=True))


@dataclass(frozen=True)
class Plan:
    spans: tuple
    radices: tuple
    bs: int

    @property
    def n(self):
        return math.prod(self.spans)


def select_params(n, b, precision):
    """plan.py:131-145 with the fallback of plan.py:121-128."""
    if n in CURATED:
        return Plan(*CURATED[n])
    spans = tuple(2 ** e for e in stage_exponents(n.bit_length() - 1))
    bpc = 8 if precision == "single" else 16
    bs = max(1, min(32, 2 ** 20 // (n * bpc)))
    return Plan(spans, tuple(min(16, s) for s in spans), bs)


def micro_lowering(radix):
    """fft_core.py:137-141: a radix 2^g is g//2 radix-4 passes then one radix-2."""
    g = radix.bit_length() - 1
    return [4] * (g // 2) + [2] * (g % 2)


def stage_lowering(span, micro):
    """fft_core.py:144-151."""
    out, rest = [], span
    while rest >= micro:
        out += micro_lowering(micro)
        rest //= micro
    if rest > 1:
        out += micro_lowering(rest)
    return out


def pass_list(plan):
    """(s, r, stage) for every executed pass; s = product of earlier radices."""
    s, out = 1, []
    for si, (span, micro) in enumerate(zip(plan.spans, plan.radices)):
        for r in stage_lowering(span, micro):
            out.append((s, r, si))
            s *= r
    return out


def base_table(s, r, dtype):
    """fft_core.py:176-182: omega_{s r}^q for q < s, f64 then cast, [0] = 1."""
    t = np.exp(1j * ((-2.0 * np.pi / (s * r)) * np.arange(s))).astype(dtype)
    t[0] = 1.0
    return t


@functools.lru_cache(maxsize=256)
def _plan_tables(s, r, dtype, inverse):
    """Tables are built once per plan in the reference (make_twiddles)."""
    t = base_table(s, r, np.dtype(dtype).type)
    t = np.conj(t) if inverse else t
    t.setflags(write=False)
    return t


# ---------------------------------------------------------------------------
# one Stockham pass — _kernels_py.py:13-45 / _kernels.pyx:19-84


def stockham_pass_np(src, dst, s, r, base, inverse):
    rows, n = src.shape
    m = n // (s * r)
    leg = src.reshape(rows, r, m, s)   # leg t of butterfly (p, q) at q + s(p + m t)
    res = dst.reshape(rows, m, r, s)   # output c at q + s(r p + c)
    if r == 2:
        u1 = leg[:, 1] * base
        np.add(leg[:, 0], u1, out=res[:, :, 0])
        np.subtract(leg[:, 0], u1, out=res[:, :, 1])
        return
    if r != 4:
        raise ValueError(f"radix {r}")
    w2 = base * base
    w3 = w2 * base
    u0, u1, u2, u3 = leg[:, 0], leg[:, 1] * base, leg[:, 2] * w2, leg[:, 3] * w3
    a, b = u0 + u2, u0 - u2
    c, d = u1 + u3, u1 - u3
    jd = d * (1j if inverse else -1j)
    np.add(a, c, out=res[:, :, 0])
    np.add(b, jd, out=res[:, :, 1])
    np.subtract(a, c, out=res[:, :, 2])
    np.subtract(b, jd, out=res[:, :, 3])


_PASS = stockham_pass_np


def ref_kernel_path():
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref")
    hits = sorted(glob.glob(os.path.join(here, "_kernels*.so")))
    return hits[0] if hits else None


def use_ref_kernel(enable=True):
    """Route passes through the reference's own compiled kernel (oracle/_ref)."""
    global _PASS
    if not enable:
        _PASS = stockham_pass_np
        return False
    path = ref_kernel_path()
    if path is None:
        return False
    spec = importlib.util.spec_from_file_location("_kernels", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    _PASS = mod.stockham_pass
    return True


# ---------------------------------------------------------------------------
# faults — fault.py:25-107


def flip_bit(value, bit):
    """fault.py:25-38: XOR one bit of the IEEE-754 pattern."""
    a = np.asarray(value)
    if a.dtype not in (np.float32, np.float64):
        a = a.astype(np.float64)
    u = np.uint32 if a.dtype == np.float32 else np.uint64
    width = a.dtype.itemsize * 8
    if not 0 <= bit < width:
        raise ValueError("bit out of range")
    return (a.view(u) ^ (u(1) << u(bit))).view(a.dtype)[()]


@dataclass
class Fault:
    transaction: int
    signal: int
    element: int
    stage: int
    part: str
    bit: int
    fired: bool = False


def strike(faults, tx_index, stage, work, row0):
    """fault.py:99-107: flip before the stage's first pass; fires once."""
    for f in faults or ():
        if f.fired or f.transaction != tx_index or f.stage != stage:
            continue
        view = work.real if f.part == "re" else work.imag
        view[f.signal - row0, f.element] = flip_bit(view[f.signal - row0, f.element], f.bit)
        f.fired = True


def transform_block(plan, precision, rows, inverse=False, faults=None, tx_index=-1, row0=0):
    """fft_core.py:255-280 for one transaction block, returns a new array."""
    dtype = DTYPES[precision]
    work = np.array(rows, dtype=dtype, copy=True)
    scratch = np.empty_like(work)
    passes = pass_list(plan)
    with np.errstate(over="ignore", invalid="ignore"):
        pi = 0
        for si in range(len(plan.spans)):
            strike(faults, tx_index, si, work, row0)
            while pi < len(passes) and passes[pi][2] == si:
                s, r, _ = passes[pi]
                _PASS(work, scratch, s, r, _plan_tables(s, r, np.dtype(dtype).str, inverse), inverse)
                work, scratch = scratch, work
                pi += 1
        if inverse:
            work *= work.real.dtype.type(1.0 / plan.n)
    return work


def transactions(b, bs):
    """fft_core.py:245-252."""
    return [(i, s, min(s + bs, b)) for i, s in enumerate(range(0, b, bs))]


def execute(x, plan, inverse=False, faults=None, workers=1):
    """fft_core.py:296-329; ``workers`` > 1 uses a thread pool over
    transactions like the reference (fft_core.py:321-326)."""
    precision = precision_of(x)
    if not np.all(np.isfinite(x.view(x.real.dtype))):
        raise ValueError("batch contains non-finite values")
    y = np.empty_like(x)
    txs = transactions(x.shape[0], plan.bs)

    def run(tx):
        i, a, b = tx
        y[a:b] = transform_block(plan, precision, x[a:b], inverse, faults, i, a)

    if workers > 1 and len(txs) > 1:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=workers) as pool:
            list(pool.map(run, txs))
    else:
        for tx in txs:
            run(tx)
    return y


# ---------------------------------------------------------------------------
# checksum building blocks — abft.py:80-190, dft_oracle.py:27-90


def roots(n, dtype, sign):
    """dft_oracle.py:27-33: trig evaluated in the working precision."""
    th = (sign * 2.0 * np.pi / n) * np.arange(n)
    if dtype == np.complex64:
        th = th.astype(np.float32)
    return np.exp(1j * th).astype(dtype, copy=False)


def gemv_checksum(e, n):
    """dft_oracle.py:72-90: e^T W accumulated row by row (the cross-check order)."""
    e = np.asarray(e)
    if e.dtype not in (np.complex64, np.complex128):
        e = e.astype(np.complex128)
    if e.shape != (n,):
        raise ValueError(f"encoding vector has length {e.shape}, expected ({n},)")
    rt = roots(n, e.dtype, -1.0)
    k = np.arange(n)
    acc = np.zeros(n, dtype=e.dtype)
    for j in range(n):
        acc += e[j] * rt[(j * k) % n]
    return acc


def dft_naive(x):
    """dft_oracle.py:36-62 (forward), blocked O(N^2) direct sums."""
    x = np.asarray(x)
    if x.dtype not in (np.complex64, np.complex128):
        x = x.astype(np.complex128)
    x2 = np.atleast_2d(x)
    n = x2.shape[1]
    rt = roots(n, x2.dtype, -1.0)
    k = np.arange(n)
    y = np.empty_like(x2)
    for j0 in range(0, n, 128):
        j = np.arange(j0, min(j0 + 128, n))
        y[:, j0:j0 + len(j)] = x2 @ rt[(j[:, None] * k[None, :]) % n].T
    return y if x.ndim == 2 else y[0]


def encoding(kind, n, precision):
    """abft.py:80-104."""
    dt = DTYPES[precision]
    k = np.arange(n)
    if kind == "ones":
        return np.ones(n, dtype=dt)
    if kind == "jou":
        return np.exp((-2j * np.pi / n) * k).astype(dt)
    if kind == "wang":
        return np.exp((-2j * np.pi / 3.0) * (k % 3)).astype(dt)
    raise ValueError(kind)


@functools.lru_cache(maxsize=16)
def left_row(kind, n, precision):
    """abft.py:116-147: e^T W; oracle DFT up to 4096, the fast path above."""
    e = encoding(kind, n, precision)
    if n <= ORACLE_CAP:
        row = dft_naive(e)
    else:
        row = execute(e[None, :].astype(DTYPES[precision]), select_params(n, 1, precision))[0]
    row = np.ascontiguousarray(row)
    row.setflags(write=False)
    return row


def detect(reference, observed, delta, floor=FLOOR):
    """abft.py:155-167."""
    if not np.isfinite(observed):
        return True, float("inf")
    div = float(abs(reference - observed) / max(abs(reference), floor, FLOOR))
    return div > delta, div


def locate(weighted, unweighted, batch=None, floor=FLOOR):
    """abft.py:170-190; returns None where the reference raises Undecodable."""
    if not (np.isfinite(weighted) and np.isfinite(unweighted)):
        return None
    if abs(unweighted) <= floor:
        return None
    with np.errstate(over="ignore", invalid="ignore"):
        ratio = complex(weighted) / complex(unweighted)
    if not np.isfinite(ratio) or abs(ratio.imag) > 0.25:
        return None
    ident = int(round(float(ratio.real)))
    if batch is not None and not 1 <= ident <= batch:
        return None
    return ident


# ---------------------------------------------------------------------------
# protected run — abft.py:342-752


@dataclass
class Stats:
    signal_sweeps: int = 0
    verifications: int = 0
    corrections: int = 0
    recomputations: int = 0
    max_divergence: float = 0.0
    events: list = field(default_factory=list)   # [tx, signal, located, divergence]


def _fft_column(plan, precision, col):
    return transform_block(plan, precision, col[None, :])[0]


class _Replay:
    """abft.py:342-551 — the serial per-transaction decision replay."""

    def __init__(self, plan, precision, src, out, delta, T, enc, stats):
        self.plan, self.precision = plan, precision
        self.src, self.out, self.delta, self.T = src, out, delta, T
        self.enc, self.stats = enc, stats
        b, n = src.shape
        self.w = np.arange(1, b + 1, dtype=RDTYPES[precision])
        self.s_in = np.zeros(n, src.dtype)
        self.s_out = np.zeros(n, src.dtype)
        self.residuals = {}
        self.pending = None
        self.seen = 0
        self.nverif = 0
        self.reports = []
        self.contrib = {}
        self.win_count = 0
        self.win_corr = False
        self.win_uncorr = False

    def recompute(self, tx):
        i, a, b = tx
        self.out[a:b] = transform_block(self.plan, self.precision, self.src[a:b], False, None, i, a)
        self.stats.recomputations += 1
        self.stats.signal_sweeps += 2 * (b - a)
        if i in self.contrib:
            self.contrib[i] = self.w[a:b] @ self.out[a:b]
            self.s_out = sum(self.contrib.values())

    def correction_column(self, p):
        """abft.py:297-317: FP32 snapshots are transformed in FP64."""
        if p["snap_in"].dtype == np.complex64:
            ref = _fft_column(self.plan, "double", p["snap_in"].astype(np.complex128))
            with np.errstate(over="ignore", invalid="ignore"):
                col = (p["snap_out"].astype(np.complex128) - ref) / p["weight"]
            return col.astype(np.complex64)
        ref = _fft_column(self.plan, self.precision, p["snap_in"])
        with np.errstate(over="ignore", invalid="ignore"):
            return (p["snap_out"] - ref) / np.float64(p["weight"])

    def usable(self, p, col):
        """abft.py:320-330."""
        if not np.all(np.isfinite(col.view(col.real.dtype))):
            return False
        n = self.plan.n
        return float(np.abs(col).max()) <= 16.0 * np.log2(n) * p["floor"] * np.sqrt(n)

    def apply_pending(self, txs, decontaminate):
        """abft.py:392-418."""
        p, self.pending = self.pending, None
        col = self.correction_column(p)
        k = p["signal"]
        if self.usable(p, col):
            self.out[k] -= col
            bad, _ = detect(p["reference"], self.out[k] @ self.enc, self.delta, p["floor"])
            if not bad:
                self.stats.corrections += 1
                if decontaminate:
                    self.s_out -= p["snap_in"].real.dtype.type(p["weight"]) * col
                self.win_corr = True
                return
        self.recompute(txs[p["tx"]])
        self.win_uncorr = True

    def feed(self, tx, c_in, c_out, floors, t_in, t_out, hits, divs, txs):
        """abft.py:422-441."""
        i, a, b = tx
        self.seen += 1
        self.win_count += 1
        self.s_in += t_in
        self.s_out = self.s_out + t_out
        self.contrib[i] = t_out
        if hits.any():
            for g in range(a, b):
                self.residuals[g] = complex(c_in[g] - c_out[g])
            trig = [(a + int(l), int(l), float(divs[a + int(l)])) for l in np.nonzero(hits)[0]]
            self.handle(tx, c_in, floors, t_in, t_out, trig, txs)
        if self.seen % self.T == 0:
            self.verify(txs)

    def handle(self, tx, c_in, floors, t_in, t_out, trig, txs):
        """abft.py:443-489."""
        i, a, b = tx
        with np.errstate(over="ignore", invalid="ignore"):
            res = sum(self.residuals[g] for g in range(a, b))
            wres = sum(self.w[g] * self.residuals[g] for g in range(a, b))
        dec = locate(wres, res, batch=len(self.w))
        decoded = None if dec is None else dec - 1
        if len(trig) > 1:
            for g, _, d in trig:
                self.stats.events.append([i, g, None, d])
            if self.pending is not None:
                self.apply_pending(txs, True)
            self.recompute(tx)
            self.win_uncorr = True
            return
        g, local, d = trig[0]
        self.stats.events.append([i, g, decoded, d])
        if self.pending is not None:
            self.apply_pending(txs, False)
            self.s_in = t_in.copy()
            self.s_out = t_out.copy()
            self.contrib = {i: t_out}
            self.win_count = 1
        self.pending = dict(signal=g, weight=float(self.w[g]), snap_in=t_in, snap_out=t_out,
                            tx=i, divergence=d, located=g, reference=complex(c_in[g]),
                            floor=float(max(floors[g], FLOOR)))

    def verify(self, txs):
        """abft.py:493-541."""
        if self.win_count == 0 and self.pending is None:
            return
        located = None
        if self.pending is not None:
            located = self.pending["located"]
            self.apply_pending(txs, True)
        ref = _fft_column(self.plan, self.precision, self.s_in)
        with np.errstate(over="ignore", invalid="ignore"):
            nrm = float(np.linalg.norm(ref))
            gdiv = float(np.linalg.norm(ref - self.s_out) / max(nrm, FLOOR))
        ghit = gdiv > self.delta
        in_window = [e for e in self.stats.events if e[1] in self.residuals]
        if ghit and not in_window and not self.win_corr and not self.win_uncorr:
            self.win_uncorr = True
        div = max([e[3] for e in in_window] + ([gdiv] if ghit else []), default=gdiv)
        trig = bool(in_window) or ghit
        self.stats.verifications += 1
        self.nverif += 1
        self.reports.append([trig, self.win_corr, self.win_uncorr and not self.win_corr,
                             located if trig else None, self.nverif - 1, float(div)])
        self.s_in[:] = 0
        self.s_out[:] = 0
        self.residuals.clear()
        self.contrib = {}
        self.win_count = 0
        self.win_corr = False
        self.win_uncorr = False

    def finish(self, txs):
        if self.seen % self.T != 0 or self.pending is not None or self.win_count:
            self.verify(txs)
        return self.reports


def _jou_variant(x):
    return 2.0 * x + np.roll(x, -1, axis=1)          # abft.py:333-334


def _jou_undo(n, dtype):
    return (2.0 + np.exp((2j * np.pi / n) * np.arange(n))).astype(dtype)   # abft.py:337-339


def signal_sums(src, out, enc, row, delta):
    """abft.py:648-665."""
    n = src.shape[1]
    with np.errstate(over="ignore", invalid="ignore"):
        c_in = src @ row
        c_out = out @ enc
        v = src.view(src.real.dtype).reshape(src.shape[0], -1)
        floors = np.sqrt(np.einsum("ij,ij->i", v, v)) / np.sqrt(n)
        div = np.abs(c_in - c_out) / np.maximum(np.abs(c_in), np.maximum(floors, FLOOR))
        bad = ~np.isfinite(c_out)
        if bad.any():
            div = np.where(bad, np.inf, div)
    return c_in, c_out, floors, div


def protected(x, plan, kind="wang", delta=None, T=1, mode="fused", faults=None,
              force_engine=False):
    """abft.py:690-752. Returns (y, Stats, reports as lists)."""
    precision = precision_of(x)
    if not np.all(np.isfinite(x.view(x.real.dtype))):
        raise ValueError("batch contains non-finite values")
    if T < 1 or mode not in ("fused", "per-transaction"):
        raise ValueError("bad group size or mode")
    if precision == "single" and x.shape[0] > MAX_SINGLE_WEIGHT:
        raise ValueError("location weights above 2^24 are not exact in single precision")
    delta = DEFAULT_DELTA[precision] if delta is None else delta
    enc = encoding(kind, plan.n, precision)
    row = left_row(kind, plan.n, precision)
    stats = Stats()
    src = _jou_variant(x) if kind == "jou" else x
    out = np.empty_like(x)
    txs = transactions(x.shape[0], plan.bs)
    for i, a, b in txs:
        out[a:b] = transform_block(plan, precision, src[a:b], False, faults, i, a)
    c_in, c_out, floors, div = signal_sums(src, out, enc, row, delta)
    hits = div > delta
    stats.signal_sweeps += 2 * x.shape[0] * (2 if mode == "per-transaction" else 1)
    stats.max_divergence = max(stats.max_divergence, float(div.max()))
    rp = _Replay(plan, precision, src, out, delta, T, enc, stats)
    if hits.any() or force_engine:
        with np.errstate(over="ignore", invalid="ignore"):
            wx = rp.w[:, None] * src
            wy = rp.w[:, None] * out
            starts = [a for _, a, _ in txs]
            if len(txs) != x.shape[0]:
                wx = np.add.reduceat(wx, starts, axis=0)
                wy = np.add.reduceat(wy, starts, axis=0)
            for j, tx in enumerate(txs):
                rp.feed(tx, c_in, c_out, floors, wx[j], wy[j],
                        hits[tx[1]:tx[2]], div, txs)
            reports = rp.finish(txs)
    else:
        reports = []
        for v, first in enumerate(range(0, len(txs), T)):
            last = min(first + T, len(txs)) - 1
            a, b = txs[first][1], txs[last][2]
            s_in = rp.w[a:b] @ src[a:b]
            s_out = rp.w[a:b] @ out[a:b]
            ref = _fft_column(plan, precision, s_in)
            gdiv = float(np.linalg.norm(ref - s_out) / max(float(np.linalg.norm(ref)), FLOOR))
            stats.verifications += 1
            reports.append([gdiv > delta, False, gdiv > delta, None, v, gdiv])
    if kind == "jou":
        out /= _jou_undo(plan.n, x.dtype)
    return out, stats, reports


def offline(x, plan, kind="wang", delta=None, faults=None):
    """abft.py:755-838: post-hoc checksums, recompute on detection (3 tries)."""
    precision = precision_of(x)
    delta = DEFAULT_DELTA[precision] if delta is None else delta
    enc = encoding(kind, plan.n, precision)
    row = left_row(kind, plan.n, precision)
    stats = Stats()
    src = _jou_variant(x) if kind == "jou" else x
    out = np.empty_like(x)
    txs = transactions(x.shape[0], plan.bs)
    for i, a, b in txs:
        out[a:b] = transform_block(plan, precision, src[a:b], False, faults, i, a)
    stats.signal_sweeps += 2 * x.shape[0]
    reports = []
    sq = np.sqrt(plan.n)
    for i, a, b in txs:
        stats.signal_sweeps += 2 * (b - a)
        with np.errstate(over="ignore", invalid="ignore"):
            c_in = src[a:b] @ row
            c_out = out[a:b] @ enc
            floors = np.sqrt(np.sum(np.abs(src[a:b]) ** 2, axis=1)) / sq
        trig = []
        for l in range(b - a):
            hit, d = detect(c_in[l], c_out[l], delta, max(floors[l], FLOOR))
            stats.max_divergence = max(stats.max_divergence, d)
            if hit:
                trig.append((a + l, l, d))
                stats.events.append([i, a + l, a + l, d])
        for g, l, d in trig:
            for _ in range(3):
                out[g:g + 1] = transform_block(plan, precision, src[g:g + 1], False, None, i, g)
                stats.recomputations += 1
                stats.signal_sweeps += 2
                if not detect(c_in[l], out[g] @ enc, delta, max(floors[l], FLOOR))[0]:
                    break
            else:
                raise RuntimeError(f"signal {g} still diverges after 3 recomputations")
        stats.verifications += 1
        reports.append([bool(trig), bool(trig), False, trig[0][0] if trig else None, i,
                        max((d for _, _, d in trig), default=0.0)])
    if kind == "jou":
        out /= _jou_undo(plan.n, x.dtype)
    return out, stats, reports


# ---------------------------------------------------------------------------
# campaign helpers — fault.py:143-160


def gaussian_batch(rng, n, b, precision):
    data = rng.standard_normal((b, n)) + 1j * rng.standard_normal((b, n))
    return data.astype(DTYPES[precision])


def draw_fault(rng, plan, b, n, precision):
    """fault.py:148-160: the uniformly random strike site of one trial."""
    signal = int(rng.integers(b))
    tx = signal // plan.bs
    return Fault(transaction=tx, signal=signal, element=int(rng.integers(n)),
                 stage=int(rng.integers(len(plan.spans))),
                 part="re" if rng.integers(2) == 0 else "im",
                 bit=int(rng.integers(32 if precision == "single" else 64)))
