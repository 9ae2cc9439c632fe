"""Fused-ABFT protected timing (C3 shape family, T = 8, 1 GiB, CUDA events)
for the library TFFT_LIB points at: one line per size, for A/B of builds."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2412_05824_b200 as tf
    from paper_2412_05824_b200 import abft as A, fft_core
    tag = os.environ.get("TAG", "prod")
    for prec in ("single", "double"):
        dt, rdt, bpc = ((torch.complex64, torch.float32, 8) if prec == "single" else (torch.complex128, torch.float64, 16))
        for logn in [int(v) for v in os.environ.get("ABFT_AB_LOGN", "10,11,12").split(",")]:
            n = 1 << logn
            b = (1 << 30) // (n * bpc)
            x = torch.randn(b * n * 2, dtype=rdt, device="cuda").view(dt).view(b, n)
            y = torch.empty_like(x)
            plan = tf.build_plan(tf.select_params(n, b, prec), prec)
            T = 8
            nwin = -(-(-(-b // plan.bs)) // T)
            sums = A._DeviceSums(b, nwin)
            ctr = fft_core._Counters()
            def run():
                A.protected_device(plan, x, y, delta=A.default_delta(prec), group_size=T, counters=ctr, sums=sums)
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                run()
            e1.record()
            torch.cuda.synchronize()
            print(f"{tag} {prec} 2^{logn} {e0.elapsed_time(e1) / 10:.4f} ms", flush=True)


main()
