# one gpurun call: targeted tests (K filter), abft_ab timings, host overhead
mkdir -p gpurun_out
ABFT_AB_LOGN=${LOGN:-9,10,11,12,13} timeout 600 python tools/abft_ab.py > gpurun_out/abft_ab.log 2>&1
cat gpurun_out/abft_ab.log
timeout 300 python tools/host_overhead.py > gpurun_out/host_overhead.log 2>&1
cat gpurun_out/host_overhead.log
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "$K" > gpurun_out/tests_q.log 2>&1
  tail -5 gpurun_out/tests_q.log
fi
