"""Time the protected transform fused vs unfused (plain transform + checksum
sweep) for a few sizes; CUDA events, 1 GiB inputs, T = 8.

    python tools/abft_ab.py
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2412_05824_b200 as tf
    from paper_2412_05824_b200 import abft as A, fft_core
    for prec in ("single", "double"):
        dt, rdt, bpc = ((torch.complex64, torch.float32, 8) if prec == "single" else (torch.complex128, torch.float64, 16))
        for logn in [int(v) for v in os.environ.get("ABFT_AB_LOGN", "9,10,11,12,13,16").split(",")]:
            n = 1 << logn
            b = (1 << 30) // (n * bpc)
            x = torch.randn(b * n * 2, dtype=rdt, device="cuda").view(dt).view(b, n)
            y = torch.empty_like(x)
            plan = tf.build_plan(tf.select_params(n, b, prec), prec)
            T = 8
            nwin = -(-(-(-b // plan.bs)) // T)
            sums = A._DeviceSums(b, nwin)
            ctr = fft_core._Counters()
            res = {}
            for mode in ("plain", "0", "1"):
                def step():
                    if mode == "plain":
                        fft_core.device_execute(plan, x, y)
                    else:
                        os.environ["TFFT_ABFT_SWEEP"] = mode
                        A.protected_device(plan, x, y, delta=A.default_delta(prec), group_size=T, counters=ctr, sums=sums)
                for _ in range(3):
                    step()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(10):
                    step()
                e1.record()
                torch.cuda.synchronize()
                res[mode] = e0.elapsed_time(e1) / 10
            os.environ.pop("TFFT_ABFT_SWEEP", None)
            print(f"{prec} n=2^{logn} bs={plan.bs} plain {res['plain']:.3f} fused {res['0']:.3f} "
                  f"({100 * (res['0'] / res['plain'] - 1):+.0f}%) sweep {res['1']:.3f} "
                  f"({100 * (res['1'] / res['plain'] - 1):+.0f}%)", flush=True)
            del x, y, sums


if __name__ == "__main__":
    main()
