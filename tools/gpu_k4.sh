#!/usr/bin/env bash
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600  > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/tests.log
tail -3 $OUT/tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > $OUT/bench.json 2> $OUT/bench.err
tail -c 2500 $OUT/bench.json
TFFT_NO_K4=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-abft --sweep 13-20 > $OUT/bench_k3.json 2> $OUT/bench_k3.err
bash tools/gpu_prof.sh "k4_fp64_n1m k4_kernel 1 1 --n 1048576 --prec double" "k4_fp64_n65536 k4_kernel 1 1 --n 65536 --prec double" "k4_fp32_n1m k4_kernel 1 1 --n 1048576 --prec single"
