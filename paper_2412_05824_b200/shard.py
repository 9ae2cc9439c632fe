"""Batch sharding over the GPUs of one box (north_star item 4).

One process per GPU. Every rank transforms a contiguous range of signals whose
boundaries fall on verification windows (T * bs signals), so each window —
and therefore every detection, correction and report — lives on exactly one
GPU and is identical to the single-GPU (and reference) window. Location
weights and event indices stay GLOBAL (w_j = j + 1 over the whole batch,
abft.py:364). The only cross-GPU traffic is the reduction of the fault
counters (signal_sweeps, verifications, corrections, recomputations, event
count: sum; max_divergence: max) — one NCCL all-reduce of a few bytes over
NVLink; the variable-length event and report lists (rare) are gathered in rank
order, which is global transaction order, so the merged RunStats and reports
equal a single-GPU run's bit for bit.
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np

from .abft import DetectionReport, RunStats, _protected
from .fft_core import SignalBatch, execute_plan


def shard_bounds(b, bs, group_size, world, rank):
    """Signal range [start, stop) of ``rank``: whole windows, balanced."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    w_sig = bs * group_size
    ntx = -(-b // bs)
    nwin = -(-ntx // group_size)
    base, extra = divmod(nwin, world)
    w0 = rank * base + min(rank, extra)
    w1 = w0 + base + (1 if rank < extra else 0)
    return min(w0 * w_sig, b), min(w1 * w_sig, b), w0


def _counters_vector(stats):
    return [stats.signal_sweeps, stats.verifications, stats.corrections, stats.recomputations,
            len(stats.events)]


def reduce_stats(stats, reports, first_window, dist, device=None):
    """Merge per-rank RunStats/reports into the global ones.

    ``dist`` is torch.distributed (initialised); counters travel in one
    all-reduce (SUM) plus one (MAX) for max_divergence — on NCCL when
    ``device`` is a CUDA device, gloo otherwise.
    """
    import torch

    dev = device if device is not None else "cpu"
    vec = torch.tensor(_counters_vector(stats), dtype=torch.int64, device=dev)
    dist.all_reduce(vec)
    mx = torch.tensor([stats.max_divergence], dtype=torch.float64, device=dev)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    world = dist.get_world_size()
    local = ([(e.transaction, e.signal, e.divergence, e.located) for e in stats.events],
             [(r.triggered, r.divergence, r.located, r.corrected, r.uncorrectable, first_window + r.verification_index)
              for r in reports])
    gathered = [None] * world
    dist.all_gather_object(gathered, local)
    from .abft import DetectionEvent

    out = RunStats(signal_sweeps=int(vec[0]), verifications=int(vec[1]), corrections=int(vec[2]),
                   recomputations=int(vec[3]), max_divergence=float(mx[0]))
    merged_reports = []
    for ev, rp in gathered:  # rank order == global transaction order
        out.events.extend(DetectionEvent(*e) for e in ev)
        merged_reports.extend(DetectionReport(*r) for r in rp)
    assert len(out.events) == int(vec[4])
    return out, merged_reports


def run_protected_sharded(plan, x_local, *, global_b, rank, world, dist, e_left="wang", delta=None,
                          group_size=1, mode="fused", injector=None, device=None, out=None):
    """run_protected on this rank's shard of a ``global_b``-signal batch.

    ``x_local`` holds exactly rows shard_bounds(...)[0:2] of the global batch.
    Returns (local output SignalBatch, global RunStats, global reports).
    """
    start, stop, w0 = shard_bounds(global_b, plan.bs, group_size, world, rank)
    batch = x_local if isinstance(x_local, SignalBatch) else SignalBatch(x_local)
    if batch.b != stop - start:
        raise ValueError(f"rank {rank} expects {stop - start} signals, got {batch.b}")
    stats = RunStats()
    y, reports = _protected(plan, batch, e_left, delta, group_size, mode, injector, stats, out, start, global_b)
    g_stats, g_reports = reduce_stats(stats, reports, w0, dist, device)
    return y, g_stats, g_reports


def execute_plan_sharded(plan, x_local, *, global_b, rank, world, direction="forward", stats=None):
    """Plain transform of this rank's contiguous shard (no collective)."""
    batch = x_local if isinstance(x_local, SignalBatch) else SignalBatch(x_local)
    return execute_plan(plan, batch, direction, stats=stats)
