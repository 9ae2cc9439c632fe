import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2412_05824_b200 as tf
from paper_2412_05824_b200 import fft_core
n = 1 << 22; b = 16
torch.manual_seed(0)
x = torch.randn(b * n * 2, dtype=torch.float64, device="cuda").view(torch.complex128).view(b, n)
ref = torch.fft.fft(x, dim=1)
y = torch.empty_like(x)
plan = tf.build_plan(tf.select_params(n, b, "double"), "double")
found = 0
for rep in range(60):
    y.zero_()
    fft_core.device_execute(plan, x, y)
    err = (y - ref).abs() > 1e-6 * ref.abs().mean()
    rows = torch.nonzero(err.any(dim=1)).flatten().tolist()
    for r in rows:
        idx = torch.nonzero(err[r]).flatten()
        q = (idx % 2048).unique(); j = (idx // 2048).unique()
        print(f"rep {rep} row {r}: {idx.numel()} bad elems; k%2048 unique {q.numel()} {q[:8].tolist()}; k//2048 unique {j.numel()} {j[:8].tolist()}", flush=True)
        found += 1
    if found >= 6: break
