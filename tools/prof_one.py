"""Run one transform configuration a few times (for ncu captures under gpurun).

    python tools/prof_one.py --n 4096 --prec double [--abft --T 8] [--reps 3]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--prec", default="double")
    ap.add_argument("--bytes", type=int, default=2 ** 30, help="input bytes")
    ap.add_argument("--abft", action="store_true")
    ap.add_argument("--T", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch
    import paper_2412_05824_b200 as tf
    from paper_2412_05824_b200 import abft as A, fft_core
    dt, rdt, bpc = ((torch.complex64, torch.float32, 8) if a.prec == "single" else (torch.complex128, torch.float64, 16))
    b = a.bytes // (a.n * bpc)
    x = torch.randn(b * a.n * 2, dtype=rdt, device="cuda").view(dt).view(b, a.n)
    y = torch.empty_like(x)
    plan = tf.build_plan(tf.select_params(a.n, b, a.prec), a.prec)
    if a.abft:
        nwin = -(-(-(-b // plan.bs)) // a.T)
        sums = A._DeviceSums(b, nwin)
        ctr = fft_core._Counters()
        for _ in range(a.reps):
            A.protected_device(plan, x, y, delta=A.default_delta(a.prec), group_size=a.T, counters=ctr, sums=sums)
    else:
        for _ in range(a.reps):
            fft_core.device_execute(plan, x, y)
    torch.cuda.synchronize()
    print("done", a.n, a.prec, b, "abft" if a.abft else "plain")


if __name__ == "__main__":
    main()
