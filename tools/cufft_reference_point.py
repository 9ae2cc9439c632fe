"""Reference point only (NOT the product, which never calls cuFFT): torch.fft
(cuFFT) on the same 1 GiB batched shapes, to calibrate what fraction of the
HBM roofline a vendor library reaches on this B200 for each N."""
import sys

import torch

peak = 6552.3
for prec in ("double", "single"):
    dt, bpc = (torch.complex128, 16) if prec == "double" else (torch.complex64, 8)
    for logn in range(8, 23):
        n = 1 << logn
        b = (1 << 30) // (n * bpc)
        x = torch.randn(b, n, dtype=dt, device="cuda")
        for _ in range(3):
            y = torch.fft.fft(x, dim=1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            y = torch.fft.fft(x, dim=1)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        gbs = 2 * n * b * bpc / (ms / 1e3) / 1e9
        print(f"cufft {prec} 2^{logn} {ms:.4f} ms frac {gbs / peak:.3f}", flush=True)
        del x, y
        torch.cuda.empty_cache()
