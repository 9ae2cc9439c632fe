"""cProfile of one injected protected call at C3 FP64 (one fault per window),
after warm-up: where the host time of the batched correction goes."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch
    import paper_2412_05824_b200 as tf
    n, b, T = 4096, 16384, 8
    plan = tf.build_plan(tf.select_params(n, b, "double"), "double")
    x = torch.randn(b, 2 * n, dtype=torch.float64, device="cuda").view(torch.complex128)
    batch = tf.SignalBatch(x)
    ntx = b // plan.bs
    nwin = ntx // T

    def call():
        inj = tf.FaultInjector(seu=False)
        for w in range(nwin):
            tx = w * T + 1
            inj.arm(tf.FaultSpec(transaction=tx, signal=tx * plan.bs, element=17, stage=0, part="re", bit=51),
                    plan=plan, batch=batch)
        stats = tf.RunStats()
        out, reports = tf.run_protected(plan, batch, group_size=T, injector=inj, stats=stats)
        torch.cuda.synchronize()
        return stats
    for _ in range(3):
        call()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(5):
        s = call()
    pr.disable()
    print("corrections", s.corrections)
    pstats.Stats(pr).sort_stats("cumulative").print_stats(30)


main()
