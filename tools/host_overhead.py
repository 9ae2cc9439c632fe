"""Wall-clock breakdown of execute_plan vs run_protected on a small host batch
(the reference's acceptance criterion 5 shape: FP32 N=1024, B=256, T=8)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2412_05824_b200 as tf
    from paper_2412_05824_b200 import abft as A, fft_core, _device
    n, b = 1024, 256
    rng = np.random.default_rng(55)
    x = (rng.standard_normal((b, n)) + 1j * rng.standard_normal((b, n))).astype(np.complex64)
    batch = tf.SignalBatch(x)
    plan = tf.build_plan(tf.select_params(n, b, "single"), "single")

    def best(fn, k=30):
        fn()
        ts = []
        for _ in range(k):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return min(ts) * 1e6

    print("execute_plan      %.1f us" % best(lambda: tf.execute_plan(plan, batch)))
    print("run_protected T=8 %.1f us" % best(lambda: tf.run_protected(plan, batch, group_size=8)))
    xd = _device.to_device(x)
    yd = torch.empty_like(xd)
    ntx = -(-b // plan.bs)
    sums = A._DeviceSums(b, -(-ntx // 8))
    ctr = fft_core._Counters()
    print("to_device         %.1f us" % best(lambda: _device.to_device(x)))
    print("device_execute    %.1f us" % best(lambda: fft_core.device_execute(plan, xd, yd, counters=ctr)))
    print("protected_device  %.1f us" % best(lambda: A.protected_device(plan, xd, yd, delta=1e-4, group_size=8,
                                                                        counters=sums.counters, sums=sums)))
    print("status read       %.1f us" % best(lambda: sums.status()))
    print("_DeviceSums alloc %.1f us" % best(lambda: A._DeviceSums(b, 32)))
    print("counters read     %.1f us" % best(lambda: ctr.read()))
    out = np.empty_like(x)
    print("D2H (_output)     %.1f us" % best(lambda: fft_core._output(batch, yd, out)))


if __name__ == "__main__":
    main()
