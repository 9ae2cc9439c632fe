"""C4 probe: FP32/FP64 N=2^22 (2 GiB in) protected runs with one injected
fault per verification window (T=2), timed end to end; --profile prints the
host-side hot spots of the replay."""
import cProfile
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_2412_05824_b200 as tf
from paper_2412_05824_b200 import fft_core


def run(prec, bpc, profile=False, logn=22, bit=None):
    n = 2 ** logn
    b = 2 ** 31 // (n * bpc)
    rdt = torch.float32 if prec == "single" else torch.float64
    cdt = torch.complex64 if prec == "single" else torch.complex128
    xd = torch.randn(b * n * 2, dtype=rdt, device="cuda").view(cdt).view(b, n)
    yd = torch.empty_like(xd)
    plan = tf.build_plan(tf.select_params(n, b, prec), prec)
    T = 2
    batch = tf.SignalBatch(xd)
    rng = np.random.default_rng(0xC4)
    inj = tf.FaultInjector(seu=False)
    nwin = -(-(-(-b // plan.bs)) // T)
    for w in range(nwin):
        tx = w * T + int(rng.integers(0, T))
        inj.arm(tf.FaultSpec(transaction=tx, signal=tx * plan.bs, element=int(rng.integers(0, n)), stage=0, part="re",
                             bit=bit if bit is not None else (30 if prec == "single" else 62)), plan=plan, batch=batch)
    fft_core.device_execute(plan, xd, yd)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fft_core.device_execute(plan, xd, yd)
    torch.cuda.synchronize()
    tp = time.perf_counter() - t0
    # first protected call pays the one-time setup (left checksum row for N =
    # 2^22 in extended precision, workspaces); the timed call is the second
    tf.run_protected(plan, batch, group_size=T, stats=tf.RunStats())
    torch.cuda.synchronize()
    stats = tf.RunStats()
    pr = cProfile.Profile() if profile else None
    t0 = time.perf_counter()
    if pr:
        pr.enable()
    out, reports = tf.run_protected(plan, batch, group_size=T, injector=inj, stats=stats)
    torch.cuda.synchronize()
    if pr:
        pr.disable()
    tq = time.perf_counter() - t0
    print(prec, n, b, "plain ms", round(tp * 1e3, 2), "protected ms", round(tq * 1e3, 1), "injections", nwin,
          "events", len(stats.events), "corrections", stats.corrections, "recomputations", stats.recomputations,
          "triggered windows", sum(r.triggered for r in reports), flush=True)
    if pr:
        pstats.Stats(pr).sort_stats("cumulative").print_stats(25)


if __name__ == "__main__":
    prof = "--profile" in sys.argv
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    logn = int(args[0]) if args else 22
    bits = (int(args[1]), int(args[2])) if len(args) > 2 else (None, None)
    run("single", 8, prof, logn, bits[0])
    run("double", 16, prof, logn, bits[1])
