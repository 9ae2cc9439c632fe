"""Host-batch (pinned) execute_plan timing, for the pipeline chunk size
(TFFT_PIPELINE_CHUNK_MB): 1 GiB FP64 batches at a few N."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import os
    import torch
    import paper_2412_05824_b200 as tf
    total = (1 << 30) // 16
    hin = torch.randn(total * 2, dtype=torch.float64).view(torch.complex128).pin_memory()
    hout = torch.empty(total, dtype=torch.complex128).pin_memory()
    xin, xout = hin.numpy(), hout.numpy()
    for logn in (10, 16, 20):
        n = 1 << logn
        plan = tf.build_plan(tf.select_params(n, total // n, "double"), "double")
        b = tf.SignalBatch(xin.reshape(-1, n))
        tf.execute_plan(plan, b, out=xout.reshape(-1, n))
        t0 = time.perf_counter()
        for _ in range(5):
            tf.execute_plan(plan, b, out=xout.reshape(-1, n))
        el = (time.perf_counter() - t0) / 5
        print(f"chunk {os.environ.get('TFFT_PIPELINE_CHUNK_MB', '64')} MB  2^{logn}: {el * 1e3:.2f} ms  "
              f"{2 * (1 << 30) / el / 1e9:.1f} GB/s (H2D + D2H)", flush=True)


main()
