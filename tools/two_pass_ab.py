"""Time the plain two-pass transforms (K7; K4 at FP32 2^21..2^22) over 1 GiB inputs for
a list of log2 N (env TP_LOGN), CUDA events, 10 reps after 3 warm-ups."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2412_05824_b200 as tf
    from paper_2412_05824_b200 import fft_core
    peak = 6552.3
    for prec in os.environ.get("TP_PREC", "double,single").split(","):
        dt, rdt, bpc = ((torch.complex64, torch.float32, 8) if prec == "single" else (torch.complex128, torch.float64, 16))
        for logn in [int(v) for v in os.environ.get("TP_LOGN", "13,14,15,16,17,18,19,20").split(",")]:
            n = 1 << logn
            b = (1 << 30) // (n * bpc)
            x = torch.randn(b * n * 2, dtype=rdt, device="cuda").view(dt).view(b, n)
            y = torch.empty_like(x)
            plan = tf.build_plan(tf.select_params(n, b, prec), prec)
            for _ in range(3):
                fft_core.device_execute(plan, x, y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                fft_core.device_execute(plan, x, y)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            gbs = 2 * n * b * bpc / (ms / 1e3) / 1e9
            print(f"{prec} 2^{logn} {ms:.4f} ms {gbs:.0f} GB/s frac {gbs / peak:.3f}", flush=True)
            del x, y


if __name__ == "__main__":
    main()
