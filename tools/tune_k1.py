"""Sweep the K1 shape variants (csrc/tfft_k1.cu kK1Var) on the B200.

    TFFT_LIB=paper_2412_05824_b200/libtfft_tune.so python tools/tune_k1.py

Prints, per (precision, N, mode), the device GB/s of every variant (1 GiB
input, CUDA events, median of 10 after 3 warm-ups).
"""
import ctypes
import os
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("TFFT_LIB", str(ROOT / "paper_2412_05824_b200" / "libtfft_tune.so"))


def main():
    import torch
    import paper_2412_05824_b200 as tf
    from paper_2412_05824_b200 import _lib, abft as A, fft_core

    lib = _lib.load()
    setv = lib.tfft_tune_set_variant
    setv.argtypes = [ctypes.c_int]
    cases = [("double", 256), ("double", 1024), ("double", 4096), ("single", 256), ("single", 1024),
             ("single", 4096), ("single", 8192)]
    out = []
    for prec, n in cases:
        dt, rdt, bpc = ((torch.complex64, torch.float32, 8) if prec == "single" else (torch.complex128, torch.float64, 16))
        b = 2 ** 30 // (n * bpc)
        x = torch.randn(b * n * 2, dtype=rdt, device="cuda").view(dt).view(b, n)
        y = torch.empty_like(x)
        plan = tf.build_plan(tf.select_params(n, b, prec), prec)
        for mode in ("plain", "abft"):
            T = 8
            nwin = -(-(-(-b // plan.bs)) // T)
            sums = A._DeviceSums(b, nwin)
            ctr = fft_core._Counters()
            ref = None
            for v in range(8):
                setv(v)

                def run():
                    if mode == "plain":
                        fft_core.device_execute(plan, x, y)
                    else:
                        A.protected_device(plan, x, y, delta=A.default_delta(prec), group_size=T, counters=ctr,
                                           sums=sums)
                try:
                    for _ in range(3):
                        run()
                    torch.cuda.synchronize()
                    ts = []
                    for _ in range(10):
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record()
                        run()
                        e1.record()
                        e1.synchronize()
                        ts.append(e0.elapsed_time(e1) / 1e3)
                    t = statistics.median(ts)
                    same = True
                    if ref is None:
                        ref = y.clone()
                    else:
                        same = bool(torch.equal(ref, y))
                    line = f"{prec:6s} n={n:5d} {mode:5s} v{v}: {2 * b * n * bpc / t / 1e9:8.1f} GB/s  {t * 1e6:8.1f} us  same={same}"
                except Exception as exc:  # noqa: BLE001
                    line = f"{prec:6s} n={n:5d} {mode:5s} v{v}: FAILED {exc}"
                print(line, flush=True)
                out.append(line)
        del x, y
        torch.cuda.empty_cache()
    setv(-1)
    (ROOT / "gpurun_out" / "tune_k1.txt").write_text("\n".join(out) + "\n")


if __name__ == "__main__":
    main()
