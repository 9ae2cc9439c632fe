"""Plain transform time with K7 vs K4 (TFFT_NO_K7) for the two-pass sizes,
1 GiB inputs, CUDA events.

    python tools/k7_ab.py [single|double]
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2412_05824_b200 as tf
    from paper_2412_05824_b200 import fft_core
    prec = sys.argv[1] if len(sys.argv) > 1 else "single"
    dt, rdt, bpc = ((torch.complex64, torch.float32, 8) if prec == "single" else (torch.complex128, torch.float64, 16))
    for logn in range(13, 21):
        n = 1 << logn
        b = (1 << 30) // (n * bpc)
        x = torch.randn(b * n * 2, dtype=rdt, device="cuda").view(dt).view(b, n)
        y = torch.empty_like(x)
        plan = tf.build_plan(tf.select_params(n, b, prec), prec)
        res = {}
        for mode in ("k7", "k4"):
            if mode == "k4":
                os.environ["TFFT_NO_K7"] = "1"
            else:
                os.environ.pop("TFFT_NO_K7", None)
            for _ in range(3):
                fft_core.device_execute(plan, x, y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                fft_core.device_execute(plan, x, y)
            e1.record()
            torch.cuda.synchronize()
            res[mode] = e0.elapsed_time(e1) / 10
        os.environ.pop("TFFT_NO_K7", None)
        gbs = 2 * n * b * bpc / res["k7"] / 1e6
        print(f"{prec} n=2^{logn} k7 {res['k7']:.3f} ms ({gbs:.0f} GB/s) k4 {res['k4']:.3f} ms", flush=True)
        del x, y


if __name__ == "__main__":
    main()
