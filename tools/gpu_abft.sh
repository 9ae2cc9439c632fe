#!/usr/bin/env bash
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/tests.log
tail -3 $OUT/tests.log
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > $OUT/bench.json 2>&1
bash tools/gpu_prof.sh "k5abft_fp32_n4096 k5_kernel 1 1 --n 4096 --prec single --abft" "k5abft_fp32_n1024 k5_kernel 1 1 --n 1024 --prec single --abft" "k5abft_fp64_n1024 k5_kernel 1 1 --n 1024 --prec double --abft" "k5_fp32_n4096 k5_kernel 1 1 --n 4096 --prec single"
