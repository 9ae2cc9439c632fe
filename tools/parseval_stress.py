"""Repeat full 1 GiB transforms and count rows whose energy breaks Parseval
(a cheap full-batch integrity check): env PS_LOGN, PS_PREC, PS_REPS, PS_INV."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2412_05824_b200 as tf
    from paper_2412_05824_b200 import fft_core
    prec = os.environ.get("PS_PREC", "double")
    dt, rdt, bpc = ((torch.complex64, torch.float32, 8) if prec == "single" else (torch.complex128, torch.float64, 16))
    tol = 1e3 * (1e-7 if prec == "single" else 1e-16)
    inv = bool(int(os.environ.get("PS_INV", "0")))  # inverse: y = x * ... / n, so Parseval scales by 1/n
    for logn in [int(v) for v in os.environ.get("PS_LOGN", "13,14,16,20").split(",")]:
        n = 1 << logn
        b = (1 << 30) // (n * bpc)
        x = torch.randn(b * n * 2, dtype=rdt, device="cuda").view(dt).view(b, n)
        y = torch.empty_like(x)
        plan = tf.build_plan(tf.select_params(n, b, prec), prec)
        ex = (x.abs() ** 2).sum(dim=1, dtype=torch.float64)
        bad = []
        for rep in range(int(os.environ.get("PS_REPS", "5"))):
            y.zero_()
            fft_core.device_execute(plan, x, y, inverse=inv)
            ey = (y.abs() ** 2).sum(dim=1, dtype=torch.float64) * (n if inv else 1.0 / n)
            err = (ey - ex).abs() / ex
            nb = int((err > tol * logn).sum())
            rows = torch.nonzero(err > tol * logn).flatten()[:8].tolist()
            bad.append((nb, rows))
        print(prec, f"2^{logn}", "bad rows per rep:", [b_[0] for b_ in bad], "first:", [b_[1] for b_ in bad if b_[0]][:3],
              flush=True)


main()
