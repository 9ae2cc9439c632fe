"""world_size-2 gloo run of the multi-GPU host path (shard.reduce_stats): the
counters are summed / maxed through one collective and the event and report
lists are gathered in rank (= global transaction) order."""

import os
import socket

import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _local_result(rank):
    from paper_2412_05824_b200.abft import DetectionEvent, DetectionReport, RunStats
    # rank r owns windows [4r, 4r+4) of 8; one event on rank 1 only
    st = RunStats(signal_sweeps=2 * 64 + (2 if rank == 1 else 0), verifications=4, corrections=rank,
                  recomputations=1 if rank == 1 else 0, max_divergence=[1e-6, 3.5][rank])
    reports = []
    for w in range(4):
        trig = rank == 1 and w == 2
        reports.append(DetectionReport(trig, 3.5 if trig else 1e-7, 70 if trig else None, trig, False, w))
    if rank == 1:
        st.events.append(DetectionEvent(transaction=70, signal=70, divergence=3.5, located=70))
    return st, reports


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2412_05824_b200.shard import reduce_stats, shard_bounds
        start, stop, w0 = shard_bounds(128, 8, 2, world, rank)
        st, reports = _local_result(rank)
        g, rep = reduce_stats(st, reports, w0, dist)
        q.put((rank, (start, stop, w0), g.signal_sweeps, g.verifications, g.corrections, g.recomputations,
               g.max_divergence, [(e.transaction, e.signal, e.located) for e in g.events],
               [(r.triggered, r.corrected, r.verification_index) for r in rep]))
    finally:
        dist.destroy_process_group()


def test_two_rank_counter_reduction_and_gather():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    results.sort()
    (_, b0, *g0), (_, b1, *g1) = results
    assert b0 == (0, 64, 0) and b1 == (64, 128, 4)
    assert g0 == g1  # every rank holds the same global view
    sweeps, verif, corr, recomp, mx, events, reports = g0
    assert (sweeps, verif, corr, recomp, mx) == (2 * 128 + 2, 8, 1, 1, 3.5)
    assert events == [(70, 70, 70)]
    assert [r[2] for r in reports] == list(range(8))
    assert [r[0] for r in reports] == [False] * 6 + [True, False]
