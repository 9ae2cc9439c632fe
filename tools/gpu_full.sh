#!/usr/bin/env bash
# one gpurun call: GPU parity tests, smoke, bench, launch list, ncu captures.
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/tests.log
tail -3 $OUT/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
tail -c 3000 $OUT/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-abft > /dev/null 2>&1
bash tools/gpu_prof.sh "k1_fp64_n4096 k1_kernel 2 1 --n 4096 --prec double" \
  "k3_fp64_n1m col_kernel 2 2 --n 1048576 --prec double" \
  "k1_fp32_n1024 k1_kernel 2 1 --n 1024 --prec single" \
  "k1abft_fp32_n4096 k1_kernel 2 1 --n 4096 --prec single --abft"
