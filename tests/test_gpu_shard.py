"""GPU-count invariance: running the batch as 1, 2, 3 or 4
window-aligned shards with global weights gives bitwise the same outputs and
the same events / counters / reports as one unsharded run. Ranks are simulated
one after another on cuda:0 (the driver's boxes have one GPU); the merge is
the one shard.reduce_stats performs over NCCL."""

import dataclasses

import numpy as np
import pytest

from conftest import gaussian

pytestmark = pytest.mark.gpu

CASES = [
    ("fp32_1024_bs1", 1024, 64, "single", 2, dict(transaction=37, signal=37, element=5, stage=0, part="re", bit=30)),
    ("fp64_4096_bs16", 4096, 64, "double", 2, dict(transaction=2, signal=40, element=77, stage=0, part="im", bit=62)),
    ("fp32_65536_k3", 65536, 12, "single", 2, dict(transaction=4, signal=9, element=4000, stage=1, part="re",
                                                   bit=30)),
]


def _merge(parts):
    from paper_2412_05824_b200.abft import RunStats
    st = RunStats()
    reports = []
    ys = []
    for y, s, rep, w0 in parts:
        ys.append(y)
        st.signal_sweeps += s.signal_sweeps
        st.verifications += s.verifications
        st.corrections += s.corrections
        st.recomputations += s.recomputations
        st.max_divergence = max(st.max_divergence, s.max_divergence)
        st.events.extend(s.events)
        reports.extend(dataclasses.replace(r, verification_index=w0 + r.verification_index) for r in rep)
    return np.concatenate(ys), st, reports


@pytest.mark.parametrize("name,n,b,precision,T,spec", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_equals_unsharded(name, n, b, precision, T, spec, world):
    import paper_2412_05824_b200 as tf
    from paper_2412_05824_b200.abft import RunStats, _protected
    from paper_2412_05824_b200.shard import shard_bounds

    x = gaussian(n, b, precision, seed=n + b)
    plan = tf.build_plan(tf.select_params(n, b, precision), precision)
    batch = tf.SignalBatch(x)
    inj = tf.FaultInjector()
    inj.arm(tf.FaultSpec(**spec), plan=plan, batch=batch)
    full_stats = RunStats()
    y_full, rep_full = tf.run_protected(plan, batch, group_size=T, injector=inj, stats=full_stats)
    parts = []
    for rank in range(world):
        s, e, w0 = shard_bounds(b, plan.bs, T, world, rank)
        if e <= s:
            continue
        inj_r = tf.FaultInjector()
        inj_r.specs.append(tf.FaultSpec(**spec))  # every rank holds the global spec list
        st = RunStats()
        y, rep = _protected(plan, tf.SignalBatch(x[s:e]), "wang", None, T, "fused", inj_r, st, None, s, b)
        parts.append((y.data, st, rep, w0))
    y, st, rep = _merge(parts)
    assert np.array_equal(y, y_full.data)
    assert [(e.transaction, e.signal) for e in st.events] == [(e.transaction, e.signal) for e in full_stats.events]
    assert (st.signal_sweeps, st.verifications, st.corrections, st.recomputations) == (
        full_stats.signal_sweeps, full_stats.verifications, full_stats.corrections, full_stats.recomputations)
    assert [(r.triggered, r.corrected, r.uncorrectable, r.verification_index) for r in rep] == [
        (r.triggered, r.corrected, r.uncorrectable, r.verification_index) for r in rep_full]
