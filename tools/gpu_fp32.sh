OUT=gpurun_out; mkdir -p $OUT
python - <<'PY' > $OUT/fp32_k4.txt 2>&1
import torch, sys
sys.path.insert(0,'.')
import paper_2412_05824_b200 as tf
from paper_2412_05824_b200 import fft_core
for n in [2**13, 2**14, 2**16, 2**18, 2**20]:
    b = 2**30 // (n*8)
    x = torch.randn(b*n*2, dtype=torch.float32, device='cuda').view(torch.complex64).view(b, n)
    y = torch.empty_like(x)
    plan = tf.build_plan(tf.select_params(n, b, 'single'), 'single')
    for _ in range(3): fft_core.device_execute(plan, x, y)
    torch.cuda.synchronize()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): fft_core.device_execute(plan, x, y)
    z.record(); torch.cuda.synchronize()
    t = a.elapsed_time(z) / 10
    print(f"fp32 n={n} ms={t:.4f} GB/s={2*2**30/t/1e6:.0f}")
PY
cat $OUT/fp32_k4.txt
