"""Real multi-process runs of the sharded path on the one GPU
the test boxes have: two ranks (gloo, both on cuda:0) each run
``run_protected_sharded`` on their window-aligned shard with an injected
fault; the merged stats/reports and the concatenated outputs are bitwise the
single-process run's (the reference's worker-count invariance,
tests/test_abft.py:513-525). The NCCL path of the one collective
(tfft_allreduce_stats through ProcessGroupNCCL's communicator) runs at
world size 1 (NCCL refuses two ranks on one GPU)."""

import hashlib
import os
import socket

import numpy as np
import pytest

from conftest import gaussian

pytestmark = pytest.mark.gpu

SPEC = dict(transaction=2, signal=70, element=300, stage=0, part="re", bit=30)
N, B, T = 4096, 96, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _summary(y, stats, reports):
    return (hashlib.sha256(np.ascontiguousarray(y).tobytes()).hexdigest(),
            [(e.transaction, e.signal) for e in stats.events],
            (stats.signal_sweeps, stats.verifications, stats.corrections, stats.recomputations),
            stats.max_divergence,
            [(r.triggered, r.corrected, r.uncorrectable, r.verification_index) for r in reports])


def _worker(rank, world, port, q, gather):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2412_05824_b200 as tf
        from paper_2412_05824_b200.shard import run_protected_sharded, shard_bounds
        x = gaussian(N, B, "single", seed=5)
        plan = tf.build_plan(tf.select_params(N, B, "single"), "single")
        s, e, _ = shard_bounds(B, plan.bs, T, world, rank)
        inj = tf.FaultInjector()
        inj.specs.append(tf.FaultSpec(**SPEC))  # every rank holds the global spec list
        xd = torch.from_numpy(np.ascontiguousarray(x[s:e])).cuda()
        y, stats, reports = run_protected_sharded(plan, tf.SignalBatch(xd), global_b=B, rank=rank, world=world,
                                                  dist=dist, group_size=T, injector=inj, gather_reports=gather)
        q.put((rank, y.data.cpu().numpy(), [(e.transaction, e.signal) for e in stats.events],
               (stats.signal_sweeps, stats.verifications, stats.corrections, stats.recomputations),
               stats.max_divergence,
               [(r.triggered, r.corrected, r.uncorrectable, r.verification_index) for r in reports]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("gather", [True, False])
def test_two_process_sharded_run_equals_single_process(gather):
    import torch.multiprocessing as mp
    import paper_2412_05824_b200 as tf
    x = gaussian(N, B, "single", seed=5)
    plan = tf.build_plan(tf.select_params(N, B, "single"), "single")
    inj = tf.FaultInjector()
    inj.arm(tf.FaultSpec(**SPEC), plan=plan, batch=tf.SignalBatch(x))
    stats = tf.RunStats()
    y_ref, rep_ref = tf.run_protected(plan, tf.SignalBatch(x), group_size=T, injector=inj, stats=stats)
    assert stats.events, "the injected fault must be detected"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, gather)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    y = np.concatenate([r[1] for r in res])
    assert np.array_equal(y, y_ref.data)
    want_rep = [(r.triggered, r.corrected, r.uncorrectable, r.verification_index) for r in rep_ref]
    for r in res:
        assert r[2] == [(e.transaction, e.signal) for e in stats.events]
        assert r[3] == (stats.signal_sweeps, stats.verifications, stats.corrections, stats.recomputations)
        assert r[4] == stats.max_divergence
        if gather:
            assert r[5] == want_rep
    if not gather:  # each rank holds its own windows, globally indexed
        assert res[0][5] + res[1][5] == want_rep


def _nccl_worker(port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_2412_05824_b200.abft import RunStats
        from paper_2412_05824_b200.shard import _nccl_comm, reduce_counters
        dist.barrier()
        st = RunStats(signal_sweeps=10, verifications=3, corrections=1, recomputations=2, max_divergence=0.25)
        comm = _nccl_comm(dist, "cuda")
        vec, mx = reduce_counters(st, dist, "cuda")
        q.put((comm is not None, vec, mx))
    finally:
        dist.destroy_process_group()


def test_nccl_counter_allreduce_through_c_abi():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    p.start()
    used_comm, vec, mx = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert used_comm, "ProcessGroupNCCL communicator not reachable: the C-ABI collective was not exercised"
    assert vec == [10, 3, 1, 2, 0] and mx == 0.25
