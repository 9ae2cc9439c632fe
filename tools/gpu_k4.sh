#!/usr/bin/env bash
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/tests.log
tail -3 $OUT/tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > $OUT/bench.json 2> $OUT/bench.err
tail -c 2500 $OUT/bench.json
bash tools/gpu_prof.sh "k4_fp64_n1m k4_kernel 1 1 --n 1048576 --prec double" "k4_fp64_n65536 k4_kernel 1 1 --n 65536 --prec double" \
  "k5_fp64_n4096 k5_kernel 1 1 --n 4096 --prec double" "k5_fp64_n1024 k5_kernel 1 1 --n 1024 --prec double" "k5_fp32_n1024 k5_kernel 1 1 --n 1024 --prec single" ${EXTRA_PROF}
