"""Small-shape invocations of every kernel route, for compute-sanitizer
(memcheck / racecheck / synccheck) under gpurun: K1 (N<=256), K5 plain and
fused ABFT, K7 (FP64 two-pass), K4 (FP32 two-pass), K3 fallback split,
reference-order multipass, the checksum sweep, the replay primitives (one
injected fault -> correction / recompute), Jou prologue/epilogue.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import paper_2412_05824_b200 as tf
    rng = np.random.default_rng(0)

    def batch(n, b, prec):
        dt = np.complex64 if prec == "single" else np.complex128
        return tf.SignalBatch((rng.standard_normal((b, n)) + 1j * rng.standard_normal((b, n))).astype(dt))

    cases = [(256, 8, "single"), (256, 8, "double"), (1024, 8, "single"), (4096, 4, "double"),
             (4096, 6, "single"), (8192, 3, "single"), (2 ** 13, 3, "double"), (2 ** 16, 3, "double"),
             (2 ** 16, 3, "single"), (2 ** 20, 2, "double"), (2 ** 22, 1, "single"), (2 ** 23, 1, "single")]
    for n, b, prec in cases:
        plan = tf.build_plan(tf.select_params(n, b, prec), prec)
        x = batch(n, b, prec)
        y = tf.execute_plan(plan, x)
        tf.execute_plan(plan, y, "inverse")
        for T in (1, 2):
            tf.run_protected(plan, x, group_size=T)
        inj = tf.FaultInjector()
        inj.arm(tf.FaultSpec(transaction=0, signal=0, element=n // 3, stage=0, part="re", bit=30 if prec == "single" else 62),
                plan=plan, batch=x)
        tf.run_protected(plan, x, group_size=1, injector=inj)
        print("ok", n, b, prec, flush=True)
    plan = tf.build_plan(tf.select_params(256, 8, "double"), "double")
    x = batch(256, 8, "double")
    tf.run_protected(plan, x, e_left="jou")
    tf.run_offline(plan, x)
    print("ok jou/offline", flush=True)


if __name__ == "__main__":
    main()
