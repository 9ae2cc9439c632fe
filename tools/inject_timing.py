"""Wall time of run_protected on a device batch, clean vs one mantissa fault
per verification window (correctable online), for C3 (N=4096, 1 GiB, T=8)
and C5 (FP32 N=2^16, 2048 signals, T=8)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def run(n, prec, b, T, bit, reps=3):
    import torch
    import paper_2412_05824_b200 as tf
    rdt, cdt = (torch.float32, torch.complex64) if prec == "single" else (torch.float64, torch.complex128)
    x = torch.randn(b * n * 2, dtype=rdt, device="cuda").view(cdt).view(b, n)
    batch = tf.SignalBatch(x)
    plan = tf.build_plan(tf.select_params(n, b, prec), prec)
    ntx = -(-b // plan.bs)
    nwin = -(-ntx // T)
    rng = np.random.default_rng(7)
    specs = []
    for w in range(nwin):
        tx = min(w * T + int(rng.integers(T)), ntx - 1)
        sig = tx * plan.bs + int(rng.integers(min(plan.bs, b - tx * plan.bs)))
        specs.append(dict(transaction=tx, signal=sig, element=int(rng.integers(n)), stage=0, part="re", bit=bit))

    def inj():
        i = tf.FaultInjector(seu=False)
        for sp in specs:
            i.arm(tf.FaultSpec(**sp), plan=plan, batch=batch)
        return i

    for _ in range(2):
        tf.run_protected(plan, batch, group_size=T)
        tf.run_protected(plan, batch, group_size=T, injector=inj())
    torch.cuda.synchronize()
    tc, ti = [], []
    for _ in range(reps):
        t0 = time.perf_counter()
        tf.run_protected(plan, batch, group_size=T)
        torch.cuda.synchronize()
        tc.append(time.perf_counter() - t0)
        st = tf.RunStats()
        j = inj()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tf.run_protected(plan, batch, group_size=T, injector=j, stats=st)
        torch.cuda.synchronize()
        ti.append(time.perf_counter() - t0)
    if "--trace" in sys.argv:  # host-side time per step of one injected call
        from paper_2412_05824_b200 import abft as A
        acc = {}

        def wrap(obj, name):
            f = getattr(obj, name)

            def g(*a, **k):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                r = f(*a, **k)
                torch.cuda.synchronize()
                acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
                return r
            setattr(obj, name, g)
            return f

        saved = [(A, n, wrap(A, n)) for n in ("protected_device", "_batched_windows", "_weighted_columns", "_output",
                                                "_prepare")]
        saved += [(A._DeviceSums, n, wrap(A._DeviceSums, n)) for n in ("status", "host", "__init__")]
        saved += [(A._ProtectedRun, n, wrap(A._ProtectedRun, n)) for n in ("__init__", "batched_window",
                                                                          "skip_clean_window", "feed", "finish")]
        j = inj()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tf.run_protected(plan, batch, group_size=T, injector=j, stats=tf.RunStats())
        torch.cuda.synchronize()
        tot = time.perf_counter() - t0
        for obj, n, f in saved:
            setattr(obj, n, f)
        print("trace total %.2f ms:" % (tot * 1e3), {k: round(v * 1e3, 3) for k, v in acc.items()}, flush=True)
    if "--profile" in sys.argv:
        import cProfile
        import pstats
        pr = cProfile.Profile()
        j = inj()
        torch.cuda.synchronize()
        pr.enable()
        tf.run_protected(plan, batch, group_size=T, injector=j, stats=tf.RunStats())
        torch.cuda.synchronize()
        pr.disable()
        pstats.Stats(pr).sort_stats("tottime").print_stats(12)
    c, i = min(tc), min(ti)
    print(f"{prec} n={n} b={b} T={T} windows={nwin} faults={len(specs)} events={len(st.events)} "
          f"corr={st.corrections} recomp={st.recomputations} clean {c * 1e3:.2f} ms injected {i * 1e3:.2f} ms "
          f"({100 * (i / c - 1):+.1f}%)", flush=True)


if __name__ == "__main__":
    if "--c3-fp32" in sys.argv:  # one config only (ncu launch lists)
        run(4096, "single", 32768, 8, 22, reps=1)
        sys.exit(0)
    run(4096, "single", 32768, 8, 22)
    run(4096, "double", 16384, 8, 51)
    run(65536, "single", 2048, 8, 22)
