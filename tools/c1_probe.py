"""C1 (FP32 N=1024, B=4096, L2 flushed) timing for the production library
and experiment builds (TFFT_LIB), plus the same kernel on a 1 GiB batch."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2412_05824_b200 as tf
    from paper_2412_05824_b200 import fft_core
    for n, b in ((1024, 4096), (1024, 131072)):
        x = torch.randn(b, 2 * n, device="cuda").view(torch.complex64)
        y = torch.empty_like(x)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        plan = tf.build_plan(tf.select_params(n, b, "single"), "single")
        for _ in range(5):
            fft_core.device_execute(plan, x, y)
        ts = []
        for _ in range(20):
            flush.fill_(1)
            if "--read-flush" in sys.argv:
                flush.view(torch.int64).sum()
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fft_core.device_execute(plan, x, y)
            z.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(z))
        ts.sort()
        print(f"n={n} b={b} median {ts[len(ts) // 2] * 1e3:.1f} us  min {ts[0] * 1e3:.1f} us", flush=True)


if __name__ == "__main__":
    main()
