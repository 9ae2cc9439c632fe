"""C4 three-stage sizes: plain vs protected (the opt-in fused stage ABFT,
TFFT_STAGE_ABFT=1, vs the default sweep route), device-resident 2 GiB inputs."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2412_05824_b200 as tf
    from paper_2412_05824_b200 import abft as A, fft_core
    for logn in (23, 24, 25):
        for prec, bpc in (("single", 8), ("double", 16)):
            n = 1 << logn
            b = (1 << 31) // (n * bpc)
            rdt, cdt = (torch.float32, torch.complex64) if prec == "single" else (torch.float64, torch.complex128)
            x = torch.randn(b * n * 2, dtype=rdt, device="cuda").view(cdt).view(b, n)
            y = torch.empty_like(x)
            plan = tf.build_plan(tf.select_params(n, b, prec), prec)
            T = 1
            nwin = -(-(-(-b // plan.bs)) // T)
            sums = A._DeviceSums(b, nwin)
            res = {}
            for mode in ("plain", "fused", "sweep"):
                def step():
                    if mode == "plain":
                        fft_core.device_execute(plan, x, y)
                    else:
                        if mode == "fused":
                            os.environ["TFFT_STAGE_ABFT"] = "1"
                        A.protected_device(plan, x, y, delta=A.default_delta(prec), group_size=T,
                                           counters=sums.counters, sums=sums)
                        os.environ.pop("TFFT_STAGE_ABFT", None)
                for _ in range(2):
                    step()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(5):
                    step()
                e1.record()
                torch.cuda.synchronize()
                res[mode] = e0.elapsed_time(e1) / 5
            print(f"{prec} 2^{logn} b={b} bs={plan.bs} plain {res['plain']:.3f} fused {res['fused']:.3f} "
                  f"({100 * (res['fused'] / res['plain'] - 1):+.0f}%) sweep {res['sweep']:.3f} "
                  f"({100 * (res['sweep'] / res['plain'] - 1):+.0f}%)", flush=True)
            del x, y, sums
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
