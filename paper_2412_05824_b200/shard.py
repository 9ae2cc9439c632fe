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


def _nccl_comm(dist, device):
    """The ncclComm_t of the default process group, when it is NCCL on a CUDA
    device (ProcessGroupNCCL._comm_ptr); None otherwise (gloo, CPU)."""
    if device is None or str(device) == "cpu" or dist.get_backend() != "nccl":
        return None
    try:
        import torch
        pg = dist.distributed_c10d._get_default_group()
        ptr = int(pg._get_backend(torch.device("cuda"))._comm_ptr())
        return ptr or None
    except Exception:
        return None


def reduce_counters(stats, dist, device=None):
    """The ONE collective of a sharded run: int64 SUM of the five counters and
    f64 MAX of max_divergence. On NCCL it is a single grouped launch through
    the library's C ABI (tfft_allreduce_stats, 48 bytes over NVLink);
    on gloo two typed torch all-reduces. Returns (counter list, max_div)."""
    import torch

    dev = device if device is not None else "cpu"
    vec = torch.tensor(_counters_vector(stats), dtype=torch.int64, device=dev)
    mx = torch.tensor([stats.max_divergence], dtype=torch.float64, device=dev)
    comm = _nccl_comm(dist, device)
    if comm is not None:
        from . import _device, _lib
        rc = _lib.load().tfft_allreduce_stats(vec.data_ptr(), int(vec.numel()), mx.data_ptr(), comm,
                                              _device.stream_handle())
        _lib.check(rc, "tfft_allreduce_stats")
    else:
        dist.all_reduce(vec)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    return [int(v) for v in vec.cpu().tolist()], float(mx.cpu()[0])


def reduce_stats(stats, reports, first_window, dist, device=None, gather_reports=True):
    """Merge per-rank RunStats/reports into the global ones.

    Counters: ``reduce_counters`` (the only per-call collective). The
    variable-length lists cross ranks only when needed: events only when the
    reduced event count is non-zero (rare), reports only with
    ``gather_reports`` (the full global list a single-GPU call would return);
    without it each rank keeps its own reports, whose ``verification_index``
    is already global. Rank order == global transaction order, so the merged
    lists equal a single-GPU run's bit for bit.
    """
    from .abft import DetectionEvent

    vec, mx = reduce_counters(stats, dist, device)
    out = RunStats(signal_sweeps=vec[0], verifications=vec[1], corrections=vec[2], recomputations=vec[3],
                   max_divergence=mx)
    local_reports = [(r.triggered, r.divergence, r.located, r.corrected, r.uncorrectable,
                      first_window + r.verification_index) for r in reports]
    local_events = [(e.transaction, e.signal, e.divergence, e.located) for e in stats.events]
    world = dist.get_world_size()
    if vec[4] > 0 or gather_reports:
        gathered = [None] * world
        dist.all_gather_object(gathered, (local_events if vec[4] > 0 else [],
                                          local_reports if gather_reports else []))
    else:
        gathered = [([], [])] * world
    merged_reports = []
    for ev, rp in gathered:
        out.events.extend(DetectionEvent(*e) for e in ev)
        merged_reports.extend(DetectionReport(*r) for r in rp)
    if not gather_reports:
        merged_reports = [DetectionReport(*r) for r in local_reports]
    assert len(out.events) == vec[4]
    return out, merged_reports


def run_protected_sharded(plan, x_local, *, global_b, rank, world, dist, e_left="wang", delta=None,
                          group_size=1, mode="fused", injector=None, device=None, out=None, gather_reports=True):
    """run_protected on this rank's shard of a ``global_b``-signal batch.

    ``x_local`` holds exactly rows shard_bounds(...)[0:2] of the global batch
    (numpy, or a CUDA tensor that stays on this rank's device).
    Returns (local output SignalBatch, global RunStats, reports: the global
    list, or this rank's windows only with ``gather_reports=False``).
    """
    start, stop, w0 = shard_bounds(global_b, plan.bs, group_size, world, rank)
    batch = x_local if isinstance(x_local, SignalBatch) else SignalBatch(x_local)
    if batch.b != stop - start:
        raise ValueError(f"rank {rank} expects {stop - start} signals, got {batch.b}")
    stats = RunStats()
    y, reports = _protected(plan, batch, e_left, delta, group_size, mode, injector, stats, out, start, global_b)
    g_stats, g_reports = reduce_stats(stats, reports, w0, dist, device, gather_reports)
    return y, g_stats, g_reports


def execute_plan_sharded(plan, x_local, *, global_b, rank, world, direction="forward", stats=None):
    """Plain transform of this rank's contiguous shard (no collective)."""
    batch = x_local if isinstance(x_local, SignalBatch) else SignalBatch(x_local)
    return execute_plan(plan, batch, direction, stats=stats)
