"""GPU parity: the CUDA path (through the C ABI) vs the reference's golden
fixtures and the pinned CPU oracle, on the same seeded inputs."""

import hashlib

import numpy as np
import pytest

from conftest import (EPS, gaussian, golden, golden_abft_outputs, golden_fft_outputs, l2_tol, max_rel_error,
                      oracle_tol, rel_l2, two_pass_group)

pytestmark = pytest.mark.gpu


def _tf():
    import paper_2412_05824_b200 as tf
    return tf


def plan_of(case):
    tf = _tf()
    return tf.build_plan(tf.PlanParams(tuple(case["spans"]), tuple(case["radices"]), case["bs"]), case["precision"])


def arm(plan, batch, specs, seu=False):
    tf = _tf()
    inj = tf.FaultInjector(seu=seu)
    for s in specs:
        inj.arm(tf.FaultSpec(**s), plan=plan, batch=batch)
    return inj


@pytest.mark.parametrize("case", golden()["fft_cases"], ids=lambda c: c["name"])
def test_transform_matches_reference(case):
    tf = _tf()
    x = gaussian(case["n"], case["b"], case["precision"], case["seed"])
    plan = plan_of(case)
    batch = tf.SignalBatch(x)
    inj = arm(plan, batch, case["faults"]) if case["faults"] else None
    y = tf.execute_plan(plan, batch, case["direction"], injector=inj).data
    ref = golden_fft_outputs()[case["name"]]
    if not case["faults"]:
        assert rel_l2(y, ref) <= l2_tol(case["precision"], case["n"])
        assert max_rel_error(y, ref) <= oracle_tol(case["precision"], case["n"])
    else:
        # a flipped exponent can make the faulted signal's bins huge; compare
        # per signal against its own scale, and the untouched rows bitwise-close
        for r in range(case["b"]):
            scale = max(np.abs(ref[r]).max(), 1e-300)
            err = np.abs(y[r] - ref[r]).max() / scale
            assert err <= 4 * oracle_tol(case["precision"], case["n"]), (r, err)


@pytest.mark.parametrize("case", golden()["abft_cases"], ids=lambda c: c["name"])
def test_protected_decisions_match_reference(case):
    tf = _tf()
    x = gaussian(case["n"], case["b"], case["precision"], case["seed"])
    plan = plan_of(case)
    batch = tf.SignalBatch(x)
    kw = dict(case["kwargs"])
    faults = kw.pop("faults", [])
    seu = kw.pop("seu", True)
    offline = kw.pop("offline", False)
    kind = kw.pop("kind", "wang")
    inj = arm(plan, batch, faults, seu=seu) if faults else None
    stats = tf.RunStats()
    if offline:
        out, reports = tf.run_offline(plan, batch, e_left=kind, injector=inj, stats=stats)
    else:
        out, reports = tf.run_protected(plan, batch, e_left=kind, group_size=kw.get("T", 1),
                                        mode=kw.get("mode", "fused"), injector=inj, stats=stats)
    r = case["result"]
    assert [(e.transaction, e.signal) for e in stats.events] == [(e[0], e[1]) for e in r["events"]]
    for e in stats.events:
        assert e.located in (None, e.signal)
    assert (stats.signal_sweeps, stats.verifications, stats.corrections, stats.recomputations) == (
        r["signal_sweeps"], r["verifications"], r["corrections"], r["recomputations"])
    assert [(x_.triggered, x_.corrected, x_.uncorrectable, x_.verification_index) for x_ in reports] == [
        (q[0], q[1], q[2], q[4]) for q in r["reports"]]
    ref = golden_abft_outputs()[case["name"]]
    assert max_rel_error(out.data, ref) <= 2 * oracle_tol(case["precision"], case["n"])


@pytest.mark.parametrize("camp", golden()["campaigns"], ids=lambda c: c["name"])
def test_campaign_fault_locations_bit_exact(camp):
    """north_star: the set of detected and corrected fault locations is bit-exact."""
    tf = _tf()
    from paper_2412_05824_b200 import fault as F
    plan = tf.build_plan(tf.select_params(camp["n"], camp["b"], camp["precision"]), camp["precision"])
    mismatches = []
    for trial, rec in enumerate(camp["trials"]):
        rng = np.random.default_rng((camp["seed"], trial))
        batch = F._gaussian_batch(rng, camp["n"], camp["b"], camp["precision"])
        spec = F._draw_spec(rng, plan, batch)
        assert dict(transaction=spec.transaction, signal=spec.signal, element=spec.element, stage=spec.stage,
                    part=spec.part, bit=spec.bit) == rec["spec"]
        inj = tf.FaultInjector()
        inj.arm(spec, plan=plan, batch=batch)
        stats = tf.RunStats()
        _, reports = tf.run_protected(plan, batch, group_size=camp["T"], injector=inj, stats=stats)
        got = ([(e.transaction, e.signal) for e in stats.events], stats.corrections, stats.recomputations,
               [(q.triggered, q.corrected, q.uncorrectable) for q in reports])
        want = ([(e[0], e[1]) for e in rec["events"]], rec["corrections"], rec["recomputations"],
                [tuple(q[:3]) for q in rec["reports"]])
        if got != want:
            mismatches.append((trial, got, want, rec["max_divergence"], stats.max_divergence))
    assert not mismatches, mismatches[:3]


@pytest.mark.parametrize("precision", ["single", "double"])
@pytest.mark.parametrize("n", [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192])
def test_oracle_equivalence_and_bitwise_protected(precision, n):
    """Reference test_fft_core.py:115-123 + test_abft.py:197-206 on the GPU."""
    tf = _tf()
    from oracle import ref_oracle as O
    b = 37
    x = gaussian(n, b, precision, seed=n + 5)
    params = tf.select_params(n, b, precision)
    plan = tf.build_plan(params, precision)
    y = tf.execute_plan(plan, tf.SignalBatch(x)).data
    ref = O.execute(x, O.select_params(n, b, precision))
    assert rel_l2(y, ref) <= l2_tol(precision, n)
    assert max_rel_error(y, ref) <= oracle_tol(precision, n)
    for T in (1, 3):
        stats = tf.RunStats()
        out, reports = tf.run_protected(plan, tf.SignalBatch(x), group_size=T, stats=stats)
        assert np.array_equal(out.data, y)
        assert not any(r.triggered for r in reports)
        ntx = -(-b // params.bs)
        assert len(reports) == -(-ntx // T)
        assert stats.max_divergence <= tf.default_delta(precision)


@pytest.mark.parametrize("precision", ["single", "double"])
@pytest.mark.parametrize("n", [256, 1024, 4096])
def test_roundtrip(precision, n):
    tf = _tf()
    x = gaussian(n, 5, precision, seed=3)
    plan = tf.build_plan(tf.select_params(n, 5, precision), precision)
    back = tf.execute_plan(plan, tf.execute_plan(plan, tf.SignalBatch(x)), "inverse").data
    assert max_rel_error(back, x) <= (1e-5 if precision == "single" else 1e-12)


def test_nonfinite_input_rejected():
    tf = _tf()
    x = gaussian(256, 3, "single", seed=1)
    x[1, 7] = np.inf
    plan = tf.build_plan(tf.select_params(256, 3, "single"), "single")
    with pytest.raises(ValueError):
        tf.execute_plan(plan, tf.SignalBatch(x))
    with pytest.raises(ValueError):
        tf.run_protected(plan, tf.SignalBatch(x))


def test_device_resident_batch_stays_on_device():
    tf = _tf()
    import torch
    x = gaussian(1024, 8, "single", seed=2)
    plan = tf.build_plan(tf.select_params(1024, 8, "single"), "single")
    xd = torch.from_numpy(x).cuda()
    y = tf.execute_plan(plan, tf.SignalBatch(xd))
    assert y.on_device
    assert np.array_equal(y.data.cpu().numpy(), tf.execute_plan(plan, tf.SignalBatch(x)).data)


def test_stockham_pass_boundary_and_butterflies():
    """The plugin kernel itself (_kernels.pyx:74-84) vs the reference's pass."""
    tf = _tf()
    from oracle import ref_oracle as O
    from paper_2412_05824_b200 import backend
    rng = np.random.default_rng(5)
    for dt in (np.complex64, np.complex128):
        for (n, s, r) in [(64, 1, 4), (64, 4, 4), (64, 16, 2), (128, 8, 4), (32, 16, 2)]:
            src = (rng.standard_normal((3, n)) + 1j * rng.standard_normal((3, n))).astype(dt)
            base = O.base_table(s, r, dt)
            for inv in (False, True):
                b = np.conj(base) if inv else base
                got = np.empty_like(src)
                backend.kernel().stockham_pass(src, got, s, r, b, inv)
                want = np.empty_like(src)
                O.stockham_pass_np(src, want, s, r, b, inv)
                assert np.abs(got - want).max() <= 8 * np.finfo(dt).eps * np.abs(want).max()
        with pytest.raises(ValueError):
            backend.kernel().stockham_pass(src, np.empty_like(src), 1, 8, O.base_table(1, 8, dt), False)
    for r in (2, 4, 8, 16, 32):
        u = rng.standard_normal(r) + 1j * rng.standard_normal(r)
        got = tf.butterfly_radix(u, r)
        ref = np.fft.fft(u)
        assert np.abs(got - ref).max() <= 8 * EPS["double"] * np.abs(ref).max()


@pytest.mark.parametrize("precision", ["single", "double"])
@pytest.mark.parametrize("log2n", [13, 14, 15, 16, 17, 18, 19, 20])
def test_two_pass_sizes_vs_oracle(precision, log2n):
    """C2-style sizes through K3 (two-pass) against the oracle, both directions."""
    tf = _tf()
    from oracle import ref_oracle as O
    n = 2 ** log2n
    b = 3 if log2n <= 17 else 1
    x = gaussian(n, b, precision, seed=log2n)
    plan = tf.build_plan(tf.select_params(n, b, precision), precision)
    y = tf.execute_plan(plan, tf.SignalBatch(x)).data
    ref = O.execute(x, O.select_params(n, b, precision))
    assert rel_l2(y, ref) <= l2_tol(precision, n)
    assert max_rel_error(y, ref) <= oracle_tol(precision, n)
    back = tf.execute_plan(plan, tf.SignalBatch(y), "inverse").data
    assert max_rel_error(back, x) <= (1e-5 if precision == "single" else 1e-12)


@pytest.mark.parametrize("precision,log2n", [("double", 14), ("double", 16), ("double", 17), ("double", 18),
                                             ("double", 20), ("double", 21), ("single", 14), ("single", 17),
                                             ("single", 20), ("single", 22)])
def test_two_pass_stage_strikes_vs_oracle(precision, log2n):
    """Stage-0 and stage-1 strikes executed inside the fused two-pass kernels
    (K7, K4; K7's tile-major ring at FP64 2^17) land on the same canonical
    intermediate as the reference's strike hook (fault.py:99-107): the struck
    transform equals the oracle's struck transform."""
    tf = _tf()
    from oracle import ref_oracle as O
    n = 2 ** log2n
    b = 3
    x = gaussian(n, b, precision, seed=log2n + 7)
    params = tf.select_params(n, b, precision)
    assert len(params.spans) == 2
    plan = tf.build_plan(params, precision)
    y_clean = tf.execute_plan(plan, tf.SignalBatch(x)).data
    bit = 52 if precision == "double" else 23  # lowest exponent bit: a factor of 2 (or 1/2)
    for stage, elem in ((0, n // 3 + 5), (1, n - 7), (1, 12345 % n)):
        sig = 1
        tx = sig // plan.bs
        inj = tf.FaultInjector(seu=False)
        inj.arm(tf.FaultSpec(transaction=tx, signal=sig, element=elem, stage=stage, part="re", bit=bit),
                plan=plan, batch=tf.SignalBatch(x))
        y = tf.execute_plan(plan, tf.SignalBatch(x), injector=inj).data
        ref = O.execute(x, O.select_params(n, b, precision), faults=[O.Fault(tx, sig, elem, stage, "re", bit)])
        assert rel_l2(y, ref) <= l2_tol(precision, n), (stage, elem)
        assert not np.array_equal(y[sig], y_clean[sig]), "the strike landed"
        others = [r for r in range(b) if r != sig]
        assert np.array_equal(y[others], y_clean[others]), "only the struck signal changes"


@pytest.mark.parametrize("precision", ["single", "double"])
def test_multipass_beyond_two_pass(precision):
    """N = 2^23 (three-stage curated plan) via the reference-order device passes."""
    tf = _tf()
    n = 2 ** 23
    x = gaussian(n, 1, precision, seed=23)
    plan = tf.build_plan(tf.select_params(n, 1, precision), precision)
    y = tf.execute_plan(plan, tf.SignalBatch(x)).data
    ref = np.fft.fft(x.astype(np.complex128), axis=1)
    assert rel_l2(y, ref) <= l2_tol(precision, n)
    back = tf.execute_plan(plan, tf.SignalBatch(y), "inverse").data
    assert max_rel_error(back, x) <= (1e-5 if precision == "single" else 1e-12)


@pytest.mark.parametrize("precision,log2n,groups", [("single", 14, 5), ("double", 16, 6), ("single", 20, 7),
                                                   ("double", 13, 4), ("double", 17, 5), ("double", 18, 5),
                                                   ("double", 19, 5), ("double", 20, 5), ("single", 19, 5),
                                                   ("single", 21, 4), ("single", 22, 3)])
def test_fused_two_pass_many_groups(precision, log2n, groups):
    """K4 (fused two-pass, L2 intermediate ring): batches spanning several
    ring cycles plus a short last group, against numpy's FFT in FP64, and
    bitwise equal to the same signals transformed alone (no cross-signal or
    cross-group leakage through the ring)."""
    tf = _tf()
    n = 2 ** log2n
    bpc = 8 if precision == "single" else 16
    g = two_pass_group(precision, n)  # ring group size (tfft_k3.cu k4_group)
    b = g * groups + max(1, g // 3)
    x = gaussian(n, b, precision, seed=log2n + 100)
    plan = tf.build_plan(tf.select_params(n, b, precision), precision)
    y = tf.execute_plan(plan, tf.SignalBatch(x)).data
    ref = np.fft.fft(x.astype(np.complex128), axis=1)
    assert rel_l2(y, ref) <= l2_tol(precision, n)
    for sel in (slice(0, 1), slice(b - 1, b), slice(g - 1, g + 1)):
        part = tf.execute_plan(plan, tf.SignalBatch(np.ascontiguousarray(x[sel]))).data
        assert np.array_equal(part, y[sel])
    back = tf.execute_plan(plan, tf.SignalBatch(y), "inverse").data
    assert max_rel_error(back, x) <= (1e-5 if precision == "single" else 1e-12)


@pytest.mark.parametrize("pinned", [True, False])
def test_host_batch_pipelined_bitwise(pinned):
    """Large host batches stream through H2D / transform / D2H in chunks
    (fft_core._execute_host_pipelined): bitwise equal to the device-resident
    transform, for pinned and pageable buffers, with a short last chunk."""
    import torch
    tf = _tf()
    from paper_2412_05824_b200 import fft_core
    n, b = 4096, 2100  # 65.6 MiB FP32 -> two chunks, the second short
    x = gaussian(n, b, "single", seed=11)
    if pinned:
        hx = torch.from_numpy(x).pin_memory()
        x = hx.numpy()
        hy = torch.empty_like(hx).pin_memory()
        out = hy.numpy()
    else:
        out = None
    plan = tf.build_plan(tf.select_params(n, b, "single"), "single")
    assert x.nbytes >= fft_core._PIPELINE_MIN_BYTES
    got = tf.execute_plan(plan, tf.SignalBatch(x), out=out).data
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    ref = tf.execute_plan(plan, tf.SignalBatch(xd)).data.cpu().numpy()
    assert np.array_equal(got, ref)
    back = tf.execute_plan(plan, tf.SignalBatch(got), "inverse").data
    assert max_rel_error(back, x) <= 1e-5


@pytest.mark.parametrize("precision,n,b", [("double", 1024, 5), ("single", 4096, 3), ("double", 65536, 3),
                                           ("single", 16384, 40), ("single", 4096, 4200)])
def test_nonfinite_input_rejected_every_kernel(precision, n, b):
    """K5, K4 and the chunked host pipeline all raise on a non-finite input
    (fft_core.py:283-306), plain and protected."""
    tf = _tf()
    x = gaussian(n, b, precision, seed=2)
    x[b - 1, n // 2] = complex(np.nan, 0.0)
    plan = tf.build_plan(tf.select_params(n, b, precision), precision)
    with pytest.raises(ValueError):
        tf.execute_plan(plan, tf.SignalBatch(x))
    with pytest.raises(ValueError):
        tf.run_protected(plan, tf.SignalBatch(x), group_size=2)
