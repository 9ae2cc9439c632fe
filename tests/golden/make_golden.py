"""Generate the golden fixtures that pin the oracle (and, through it, the CUDA path).

Run HERE (the container that has the read-only reference mounted); the GPU box
never imports the reference. The fixtures it writes are committed:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every fixture is produced by calling the reference package's own public API
(``resilient_fft`` from /root/reference/pkg/src, numpy backend) on seeded
inputs. Inputs are regenerated from their seeds by the tests (numpy's PCG64 +
ziggurat normal stream is stable), and a SHA-256 of each input is stored so a
drifting generator is caught instead of silently changing the fixture.
"""

from __future__ import annotations

import dataclasses
import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent

sys.dont_write_bytecode = True
sys.path.insert(0, REF_SRC)
os.environ.setdefault("RESILIENT_FFT_BACKEND", "python")

import resilient_fft as rf  # noqa: E402
from resilient_fft import abft as rabft  # noqa: E402
from resilient_fft import fault as rfault  # noqa: E402
from resilient_fft.plan import PlanParams  # noqa: E402

DT = {"single": np.complex64, "double": np.complex128}


def gaussian(n, b, precision, seed):
    rng = np.random.default_rng(seed)
    data = rng.standard_normal((b, n)) + 1j * rng.standard_normal((b, n))
    return data.astype(DT[precision])


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def plan_of(spans, radices, bs, precision):
    return rf.build_plan(PlanParams(tuple(spans), tuple(radices), bs), precision)


def spec_dict(s):
    return dict(transaction=s.transaction, signal=s.signal, element=s.element,
                stage=s.stage, part=s.part, bit=s.bit)


def arm(plan, batch, specs, seu=True):
    inj = rf.FaultInjector(seu=seu)
    for s in specs:
        inj.arm(rf.FaultSpec(**s), plan=plan, batch=batch)
    return inj


# ----------------------------------------------------------------------------
# 1. plain / faulted transforms


def fft_cases():
    cases = []
    arrays = {}

    def add(name, n, b, precision, seed, params, direction="forward", faults=()):
        x = gaussian(n, b, precision, seed)
        plan = plan_of(params.spans, params.radices, params.bs, precision)
        batch = rf.SignalBatch(x)
        inj = arm(plan, batch, faults, seu=False) if faults else None
        y = rf.execute_plan(plan, batch, direction, injector=inj).data
        cases.append(dict(name=name, n=n, b=b, precision=precision, seed=seed,
                          spans=list(params.spans), radices=list(params.radices),
                          bs=params.bs, direction=direction, faults=list(faults),
                          x_digest=digest(x)))
        arrays[name] = y

    for precision in ("single", "double"):
        for log2n in range(1, 13):
            n = 2 ** log2n
            add(f"sel_{precision}_{n}", n, 3, precision, 100 + log2n,
                rf.select_params(n, 3, precision))
        for n in (8, 256, 1024, 4096):
            add(f"inv_{precision}_{n}", n, 2, precision, 200 + n,
                rf.select_params(n, 2, precision), direction="inverse")
        add(f"two_stage_{precision}_16384", 2 ** 14, 2, precision, 314,
            rf.select_params(2 ** 14, 2, precision))
    add("curated_single_131072", 2 ** 17, 1, "single", 17,
        rf.select_params(2 ** 17, 1, "single"))
    custom = [
        ("custom_64_16x4", 64, PlanParams((16, 4), (4, 4), 1)),
        ("custom_256_8x4x8", 256, PlanParams((8, 4, 8), (8, 4, 8), 1)),
        ("custom_256_16x16", 256, PlanParams((16, 16), (16, 16), 1)),
        ("custom_2048_16x8x16", 2048, PlanParams((16, 8, 16), (16, 8, 16), 2)),
        ("custom_512_2x256", 512, PlanParams((2, 256), (2, 16), 4)),
    ]
    for name, n, params in custom:
        for precision in ("single", "double"):
            add(f"{name}_{precision}", n, 3, precision, n + 7, params)
    # in-stage strikes: they pin the canonical stage-boundary layout
    strikes = [
        ("strike_256_16x16_s1", 256, PlanParams((16, 16), (16, 16), 1), "double",
         [dict(transaction=1, signal=1, element=37, stage=1, part="re", bit=62)]),
        ("strike_256_16x16_s1_im", 256, PlanParams((16, 16), (16, 16), 1), "single",
         [dict(transaction=2, signal=2, element=200, stage=1, part="im", bit=30)]),
        ("strike_2048_3st_s2", 2048, PlanParams((16, 8, 16), (16, 8, 16), 2), "double",
         [dict(transaction=0, signal=1, element=1500, stage=2, part="re", bit=63)]),
        ("strike_2048_3st_s1", 2048, PlanParams((16, 8, 16), (16, 8, 16), 2), "single",
         [dict(transaction=1, signal=2, element=5, stage=1, part="im", bit=29)]),
        ("strike_1024_s0", 1024, PlanParams((1024,), (8,), 1), "single",
         [dict(transaction=0, signal=0, element=0, stage=0, part="re", bit=31)]),
        ("strike_16384_s1", 2 ** 14, PlanParams((128, 128), (16, 16), 4), "double",
         [dict(transaction=0, signal=1, element=9000, stage=1, part="re", bit=55)]),
    ]
    for name, n, params, precision, faults in strikes:
        add(name, n, 3, precision, n + 11, params, faults=faults)
    return cases, arrays


# ----------------------------------------------------------------------------
# 2. protected runs


def run_case(plan, x, *, T=1, kind="wang", faults=(), seu=True, mode="fused",
             offline=False, delta=None):
    batch = rf.SignalBatch(x)
    inj = arm(plan, batch, faults, seu=seu) if faults else None
    stats = rf.RunStats()
    if offline:
        out, reports = rf.run_offline(plan, batch, e_left=kind, delta=delta,
                                      injector=inj, stats=stats)
    else:
        out, reports = rf.run_protected(plan, batch, e_left=kind, delta=delta,
                                        group_size=T, mode=mode, injector=inj,
                                        stats=stats)
    rec = dict(
        events=[[e.transaction, e.signal, e.located, e.divergence] for e in stats.events],
        signal_sweeps=stats.signal_sweeps,
        verifications=stats.verifications,
        corrections=stats.corrections,
        recomputations=stats.recomputations,
        max_divergence=stats.max_divergence,
        reports=[[r.triggered, r.corrected, r.uncorrectable, r.located,
                  r.verification_index, r.divergence] for r in reports],
    )
    return out.data, rec


def abft_cases():
    cases = []
    arrays = {}

    def add(name, n, b, precision, seed, params, store_output=True, **kw):
        x = gaussian(n, b, precision, seed)
        plan = plan_of(params.spans, params.radices, params.bs, precision)
        y, rec = run_case(plan, x, **kw)
        kw = dict(kw)
        kw["faults"] = list(kw.get("faults", ()))
        cases.append(dict(name=name, n=n, b=b, precision=precision, seed=seed,
                          spans=list(params.spans), radices=list(params.radices),
                          bs=params.bs, x_digest=digest(x), kwargs=kw, result=rec))
        if store_output:
            arrays[name] = y

    P256 = lambda bs: PlanParams((256,), (16,), bs)  # noqa: E731
    for T in (1, 3):
        add(f"clean_T{T}", 256, 8, "single", 3, P256(2), T=T)
    for T in (1, 2, 3, 4, 8):
        add(f"count_T{T}", 256, 8, "single", 3, P256(2), T=T)
    for trial in range(20):
        rng = np.random.default_rng((99, trial))
        tx = int(rng.integers(2))
        sig = int(rng.integers(8))
        el = int(rng.integers(256))
        part = "re" if rng.integers(2) == 0 else "im"
        bit = int(rng.integers(32))
        sig = tx * 4 + int(rng.integers(4))
        add(f"single_fault_{trial}", 256, 8, "single", 17, P256(4),
            faults=[dict(transaction=tx, signal=sig, element=el, stage=0, part=part, bit=bit)])
    for T in (1, 2, 4, 8):
        add(f"cross_T{T}", 256, 8, "single", 23, P256(1), T=T,
            faults=[dict(transaction=5, signal=5, element=100, stage=0, part="re", bit=30)])
    add("two_faults_diff_tx", 256, 8, "single", 29, P256(1), T=8, seu=False,
        faults=[dict(transaction=1, signal=1, element=10, stage=0, part="re", bit=31),
                dict(transaction=5, signal=5, element=20, stage=0, part="im", bit=31)])
    add("two_faults_same_tx", 256, 8, "single", 31, P256(4), seu=False,
        faults=[dict(transaction=0, signal=0, element=10, stage=0, part="re", bit=31),
                dict(transaction=0, signal=2, element=20, stage=0, part="im", bit=31)])
    add("inf_fault", 256, 8, "single", 37, P256(1),
        faults=[dict(transaction=2, signal=2, element=7, stage=0, part="im", bit=30)])
    for mode in ("fused", "per-transaction"):
        add(f"mode_{mode}", 256, 8, "single", 43, P256(2), mode=mode,
            faults=[dict(transaction=1, signal=3, element=9, stage=0, part="re", bit=31)])
    add("offline_clean", 256, 8, "single", 47, P256(2), offline=True)
    add("offline_fault", 256, 8, "single", 53, P256(2), offline=True,
        faults=[dict(transaction=2, signal=4, element=11, stage=0, part="re", bit=31)])
    add("jou_clean", 256, 8, "double", 67, PlanParams((256,), (16,), 2), kind="jou")
    add("jou_fault_s1", 256, 8, "double", 71, PlanParams((16, 16), (16, 16), 1),
        kind="jou", faults=[dict(transaction=3, signal=3, element=250, stage=1, part="re", bit=52)])
    for kind in ("jou", "wang", "ones"):
        add(f"blind_{kind}", 256, 8, "double", 72, PlanParams((256,), (16,), 8), kind=kind,
            faults=[dict(transaction=0, signal=3, element=50, stage=0, part="re", bit=61)])
    # window restarts: a second fault while one is pending, inside one window
    add("restart_window", 512, 16, "single", 81, PlanParams((512,), (16,), 2), T=4, seu=False,
        faults=[dict(transaction=0, signal=1, element=3, stage=0, part="re", bit=30),
                dict(transaction=2, signal=4, element=77, stage=0, part="im", bit=31)])
    add("restart_window_fp64", 512, 16, "double", 82, PlanParams((512,), (16,), 2), T=4, seu=False,
        faults=[dict(transaction=1, signal=2, element=3, stage=0, part="re", bit=62),
                dict(transaction=3, signal=7, element=77, stage=0, part="im", bit=63)])
    # multi-stage plans with stage>=1 strikes under protection
    add("stage1_2st_fp64", 2 ** 14, 4, "double", 91, PlanParams((128, 128), (16, 16), 1), T=2,
        faults=[dict(transaction=2, signal=2, element=4321, stage=1, part="im", bit=60)])
    add("stage1_2st_fp32", 2 ** 14, 4, "single", 92, PlanParams((128, 128), (16, 16), 2), T=1,
        faults=[dict(transaction=1, signal=3, element=999, stage=1, part="re", bit=31)])
    add("stage2_3st_fp64", 2048, 6, "double", 93, PlanParams((16, 8, 16), (16, 8, 16), 2), T=2,
        faults=[dict(transaction=1, signal=3, element=1111, stage=2, part="re", bit=61)])
    return cases, arrays


def campaign_cases():
    """Seeded _draw_spec trials: the decision-parity workload."""
    out = []
    configs = [
        ("fp32_4096_b64_T2", 4096, 64, "single", 2, 0xA1, 60),
        ("fp64_4096_b64_T2", 4096, 64, "double", 2, 0xA2, 60),
        ("fp32_1024_b16_T2", 1024, 16, "single", 2, 0xA3, 80),
        ("fp32_256_b8_T1", 256, 8, "single", 1, 0xA4, 80),
        ("fp64_512_b8_T4", 512, 8, "double", 4, 0xA5, 60),
        ("fp64_16384_b4_T1", 2 ** 14, 4, "double", 1, 0xA6, 30),
        ("fp32_16384_b4_T2", 2 ** 14, 4, "single", 2, 0xA7, 30),
    ]
    for name, n, b, precision, T, seed, trials in configs:
        params = rf.select_params(n, b, precision)
        plan = rf.build_plan(params, precision)
        recs = []
        for trial in range(trials):
            rng = np.random.default_rng((seed, trial))
            batch = rfault._gaussian_batch(rng, n, b, precision)
            spec = rfault._draw_spec(rng, plan, batch)
            _, rec = run_case(plan, batch.data, T=T, faults=[spec_dict(spec)])
            rec["spec"] = spec_dict(spec)
            rec["x_digest"] = digest(batch.data)
            recs.append(rec)
        out.append(dict(name=name, n=n, b=b, precision=precision, T=T, seed=seed,
                        spans=list(params.spans), radices=list(params.radices),
                        bs=params.bs, trials=recs))
    return out


def roc_case():
    cfg = rf.CampaignConfig(total_runs=120, injected_fraction=0.5, n=256, b=4,
                            precision="single",
                            delta_sweep=(1e-7, 1e-6, 1e-5, 1e-4, 1e-3, 1e-2, 1e-1),
                            seed=1234)
    res = rf.roc_campaign(cfg)
    return dict(config=dataclasses.asdict(cfg), rows=[list(r) for r in res.rows],
                trials=[dataclasses.asdict(t) for t in res.trials])


# ----------------------------------------------------------------------------
# 3. known-answer tables


def kats():
    k = {}
    k["flip_bit_single"] = [
        [v, b, float(rf.flip_bit(np.float32(v), b))]
        for v in (1.0, -3.25, 1.5, 1e-30, 0.0) for b in (0, 7, 22, 23, 30, 31)
    ]
    k["flip_bit_double"] = [
        [v, b, float(rf.flip_bit(np.float64(v), b))]
        for v in (1.0, -3.25, 1.5, 1e-300, 0.0) for b in (0, 7, 51, 52, 62, 63)
    ]
    k["select_params"] = []
    for precision in ("single", "double"):
        for log2n in range(1, 30):
            p = rf.select_params(2 ** log2n, 1, precision)
            k["select_params"].append([precision, 2 ** log2n, list(p.spans),
                                       list(p.radices), p.bs])
    k["passes"] = []
    for params in (PlanParams((1024,), (8,), 1), PlanParams((256, 512), (16, 16), 8),
                   PlanParams((256, 128, 256), (16, 16, 16), 16), PlanParams((2, 256), (2, 16), 4),
                   PlanParams((4096,), (16,), 1), PlanParams((32,), (32,), 1)):
        plan = rf.build_plan(params, "double")
        k["passes"].append([list(params.spans), list(params.radices),
                            [[p.s, p.r, p.stage] for p in plan.passes]])
    k["left_rows"] = {}
    for kind in ("wang", "ones", "jou"):
        for precision in ("single", "double"):
            for n in (2, 4, 8, 64):
                row = rf.precompute_left(kind, n, precision).values
                k["left_rows"][f"{kind}_{precision}_{n}"] = [[float(z.real), float(z.imag)] for z in row]
    k["locate"] = [[4.0, 0, 2.0, 0, None, 2], [6e-3, 6e-3, 1e-3, 1e-3, None, 6]]
    k["detect"] = []
    for ref, obs, delta, floor in ((1.5 + 0.5j, 1.5 + 0.5j, 1e-4, 1e-30),
                                   (1.0, 1.0 - 1e-2, 1e-4, 1e-30),
                                   (0.0, 1e-8, 1e-4, 1.0),
                                   (2.0 + 1j, 2.0 + 1.0001j, 1e-5, 1e-30)):
        hit, div = rf.detect(ref, obs, delta, floor)
        k["detect"].append([[ref.real if isinstance(ref, complex) else ref,
                             ref.imag if isinstance(ref, complex) else 0.0],
                            [complex(obs).real, complex(obs).imag], delta, floor, hit, div])
    return k


def main():
    fc, fa = fft_cases()
    ac, aa = abft_cases()
    camp = campaign_cases()
    payload = dict(
        generator="tests/golden/make_golden.py",
        reference="resilient-fft " + rf.__version__ + " (numpy backend)",
        fft_cases=fc, abft_cases=ac, campaigns=camp, roc=roc_case(), kats=kats(),
    )
    (HERE / "golden.json").write_text(json.dumps(payload, indent=0, default=float))
    np.savez_compressed(HERE / "fft_outputs.npz", **fa)
    np.savez_compressed(HERE / "abft_outputs.npz", **aa)
    print("wrote", len(fc), "fft cases,", len(ac), "abft cases,",
          sum(len(c["trials"]) for c in camp), "campaign trials")


if __name__ == "__main__":
    main()
