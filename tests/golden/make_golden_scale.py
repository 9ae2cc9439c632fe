"""Reference-generated fixtures at the BASELINE config scales (C3, C4, C5) and
the reference's own acceptance protocols (ROC, criterion 4).

Run HERE (the reference is read-only under /root/reference; the GPU box never
imports it). Output is committed:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_scale.py

Everything comes from calling ``resilient_fft`` (numpy backend) on seeded
inputs; inputs are regenerated from their seeds by the tests and pinned by a
SHA-256 digest. Sections:

* ``campaigns`` — single-fault decision parity at C3 (N=4096, FP32 B=1024 /
  FP64 B=512, T=8), C5 (FP32 N=2^16, B=64, T=8), C4 (FP32/FP64 N=2^22
  (2048,2048) and N=2^23 curated (256,128,256) bs=16, stage-0/1/2 strikes).
  Half the trials use ``fault._draw_spec`` as is (fault.py:148-160), half
  redraw the bit from the exponent field so the correction / recompute paths
  are exercised at scale.
* ``multi`` — one injection per verification window in one run (C3 FP32
  B=2048 T=8: 8 windows; C4 FP32 2^22 B=8 T=1 and FP64 2^22 B=4 T=1).
* ``roc`` — the full 2000-run ROC protocol of tests/test_acceptance.py:77-110
  (n=512, b=4, seed 0x5EED), per-trial flags and the swept rows.
* ``criterion4`` — tests/test_acceptance.py:113-163 (seeds (0xC4, n, trial),
  n=2^10 and n=2^17, all 200 trials each), events at T=1.
* ``left_rows_single`` (npz) — the reference's FP32 wang rows at n = 1024,
  4096 (oracle GEMV path) and 8192, 65536 (FP32 FFT path), abft.py:116-147.
"""

from __future__ import annotations

import dataclasses
import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, REF_SRC)
os.environ.setdefault("RESILIENT_FFT_BACKEND", "python")

import resilient_fft as rf  # noqa: E402
from resilient_fft import fault as rfault  # noqa: E402
from resilient_fft.plan import PlanParams  # noqa: E402

EXP_BITS = {"single": (23, 31), "double": (52, 63)}


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def spec_dict(s):
    return dict(transaction=s.transaction, signal=s.signal, element=s.element, stage=s.stage, part=s.part,
                bit=s.bit)


def record(stats, reports):
    return dict(
        events=[[e.transaction, e.signal, e.located, e.divergence] for e in stats.events],
        signal_sweeps=stats.signal_sweeps, verifications=stats.verifications, corrections=stats.corrections,
        recomputations=stats.recomputations, max_divergence=stats.max_divergence,
        reports=[[r.triggered, r.corrected, r.uncorrectable, r.located, r.verification_index, r.divergence]
                 for r in reports])


def campaign(name, n, b, precision, T, seed, trials, params=None):
    params = params or rf.select_params(n, b, precision)
    plan = rf.build_plan(params, precision)
    recs = []
    t0 = time.time()
    for trial in range(trials):
        rng = np.random.default_rng((seed, trial))
        batch = rfault._gaussian_batch(rng, n, b, precision)
        spec = rfault._draw_spec(rng, plan, batch)
        if trial % 2 == 1:  # exponent-field bit: a strong fault
            lo, hi = EXP_BITS[precision]
            spec = dataclasses.replace(spec, bit=int(np.random.default_rng((seed, trial, 7)).integers(lo, hi)))
        inj = rf.FaultInjector()
        inj.arm(dataclasses.replace(spec, fired=False), plan=plan, batch=batch)
        stats = rf.RunStats()
        _, reports = rf.run_protected(plan, batch, group_size=T, injector=inj, stats=stats)
        rec = record(stats, reports)
        rec["spec"] = spec_dict(spec)
        rec["x_digest"] = digest(batch.data)
        recs.append(rec)
    print(f"  {name}: {trials} trials, {sum(bool(r['events']) for r in recs)} with events, "
          f"{time.time() - t0:.1f}s", flush=True)
    return dict(name=name, n=n, b=b, precision=precision, T=T, seed=seed, spans=list(params.spans),
                radices=list(params.radices), bs=params.bs, trials=recs)


def multi(name, n, b, precision, T, seed):
    """One strong fault per verification window, all armed in one run."""
    params = rf.select_params(n, b, precision)
    plan = rf.build_plan(params, precision)
    rng = np.random.default_rng(seed)
    batch = rfault._gaussian_batch(rng, n, b, precision)
    txs = rf.transaction_partition(plan, batch)
    ntx = len(txs)
    specs = []
    for w in range(-(-ntx // T)):
        r = np.random.default_rng((seed, w))
        tx = txs[min(w * T + int(r.integers(T)), ntx - 1)]
        signal = tx.start + int(r.integers(tx.stop - tx.start))
        lo, hi = EXP_BITS[precision]
        specs.append(dict(transaction=tx.index, signal=signal, element=int(r.integers(n)),
                          stage=int(r.integers(len(plan.stages))), part="re" if r.integers(2) == 0 else "im",
                          bit=int(r.integers(lo, hi))))
    inj = rf.FaultInjector(seu=False)
    for s in specs:
        inj.arm(rf.FaultSpec(**s), plan=plan, batch=batch)
    stats = rf.RunStats()
    t0 = time.time()
    out, reports = rf.run_protected(plan, batch, group_size=T, injector=inj, stats=stats)
    rec = record(stats, reports)
    rec["ref_err"] = repair_errors(plan, batch, out)
    print(f"  multi {name}: {len(specs)} faults, {len(stats.events)} events, {time.time() - t0:.1f}s", flush=True)
    return dict(name=name, n=n, b=b, precision=precision, T=T, seed=seed, spans=list(params.spans),
                radices=list(params.radices), bs=params.bs, specs=specs, x_digest=digest(batch.data), result=rec)


def repair_errors(plan, batch, out):
    """Per-signal max |protected - clean| / max |clean| of the reference itself:
    with several repaired faults in one run the FP32 correction residual can
    exceed the single-fault bound of tests/test_acceptance.py:133-156."""
    clean = rf.execute_plan(plan, batch).data
    scale = np.maximum(np.abs(clean).max(axis=1), 1e-30)
    return [float(v) for v in np.abs(out.data - clean).max(axis=1) / scale]


def add_repair_errors():
    """Augment an existing golden_scale.json with ``ref_err`` for the multi cases."""
    path = HERE / "golden_scale.json"
    payload = json.loads(path.read_text())
    for case in payload["multi"]:
        params = PlanParams(tuple(case["spans"]), tuple(case["radices"]), case["bs"])
        plan = rf.build_plan(params, case["precision"])
        batch = rfault._gaussian_batch(np.random.default_rng(case["seed"]), case["n"], case["b"], case["precision"])
        assert digest(batch.data) == case["x_digest"]
        inj = rf.FaultInjector(seu=False)
        for s in case["specs"]:
            inj.arm(rf.FaultSpec(**s), plan=plan, batch=batch)
        out, _ = rf.run_protected(plan, batch, group_size=case["T"], injector=inj, stats=rf.RunStats())
        case["result"]["ref_err"] = repair_errors(plan, batch, out)
        print(f"  {case['name']}: max ref_err {max(case['result']['ref_err']):.3g}", flush=True)
    path.write_text(json.dumps(payload, indent=0, default=float))


def roc_full():
    cfg = rf.CampaignConfig(total_runs=2000, injected_fraction=0.5, n=512, b=4, precision="single",
                            delta_sweep=(1e-7, 1e-6, 1e-5, 1e-4, 1e-3, 1e-2, 1e-1), seed=0x5EED)
    t0 = time.time()
    res = rf.roc_campaign(cfg)
    print(f"  roc: {len(res.trials)} trials, {time.time() - t0:.1f}s", flush=True)
    return dict(config=dataclasses.asdict(cfg), rows=[list(r) for r in res.rows],
                trials=[[t.injected, t.bit, t.divergence, t.detected, t.located_ok, t.corrected, t.final_ok]
                        for t in res.trials])


def criterion4_runs(n, trials):
    if n == 2 ** 10:
        params = rf.select_params(n, 8, "single")
    else:
        base = rf.select_params(n, 8, "single")
        params = PlanParams(base.spans, base.radices, bs=2)
    plan = rf.build_plan(params, "single")
    b = 8
    # reference tests/conftest.py gaussian_batch(n, b, precision, seed)
    rng = np.random.default_rng(n % 7919)
    data = (rng.standard_normal((b, n)) + 1j * rng.standard_normal((b, n))).astype(np.complex64)
    batch = rf.SignalBatch(data)
    recs = []
    t0 = time.time()
    for trial in range(trials):
        rng = np.random.default_rng((0xC4, n, trial))
        proto = rfault._draw_spec(rng, plan, batch)
        inj = rf.FaultInjector()
        inj.arm(dataclasses.replace(proto, fired=False), plan=plan, batch=batch)
        stats = rf.RunStats()
        _, reports = rf.run_protected(plan, batch, group_size=1, injector=inj, stats=stats, workers=1)
        rec = record(stats, reports)
        rec["spec"] = spec_dict(proto)
        recs.append(rec)
    print(f"  criterion4 n={n}: {trials} trials, {sum(bool(r['events']) for r in recs)} detected, "
          f"{time.time() - t0:.1f}s", flush=True)
    return dict(n=n, b=b, spans=list(params.spans), radices=list(params.radices), bs=params.bs,
                x_digest=digest(data), trials=recs)


def left_rows():
    rows = {}
    for n in (1024, 4096, 8192, 65536):
        rows[f"wang_single_{n}"] = rf.precompute_left("wang", n, "single").values
        rows[f"wang_double_{n}"] = rf.precompute_left("wang", n, "double").values
    return rows


def main():
    t0 = time.time()
    camps = [
        campaign("C3_fp32_4096_b1024_T8", 4096, 1024, "single", 8, 0xC3A, 16),
        campaign("C3_fp64_4096_b512_T8", 4096, 512, "double", 8, 0xC3B, 16),
        campaign("C5_fp32_65536_b64_T8", 2 ** 16, 64, "single", 8, 0xC5, 16),
        campaign("C4_fp32_2p22_b2_T1", 2 ** 22, 2, "single", 1, 0xC4A, 8),
        campaign("C4_fp64_2p22_b2_T1", 2 ** 22, 2, "double", 1, 0xC4B, 8),
        campaign("C4_fp32_2p23_b4_T1", 2 ** 23, 4, "single", 1, 0xC4C, 6),
        campaign("C4_fp64_2p23_b4_T1", 2 ** 23, 4, "double", 1, 0xC4D, 6),
    ]
    multis = [
        multi("C3_fp32_4096_b2048_T8", 4096, 2048, "single", 8, 0x3C3),
        multi("C4_fp32_2p22_b8_T1", 2 ** 22, 8, "single", 1, 0x4C4),
        multi("C4_fp64_2p22_b4_T1", 2 ** 22, 4, "double", 1, 0x4C5),
    ]
    payload = dict(generator="tests/golden/make_golden_scale.py",
                   reference="resilient-fft " + rf.__version__ + " (numpy backend)",
                   campaigns=camps, multi=multis, roc=roc_full(),
                   criterion4=[criterion4_runs(2 ** 10, 200), criterion4_runs(2 ** 17, 200)])
    (HERE / "golden_scale.json").write_text(json.dumps(payload, indent=0, default=float))
    np.savez_compressed(HERE / "golden_scale_rows.npz", **left_rows())
    print(f"done in {time.time() - t0:.0f}s")


if __name__ == "__main__":
    if "--repair-errors" in sys.argv:
        add_repair_errors()
    else:
        main()
