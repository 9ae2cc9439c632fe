#!/usr/bin/env bash
OUT=gpurun_out
mkdir -p $OUT
python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -m gpu -q -x --timeout 900 > $OUT/tests.log 2>&1
tail -5 $OUT/tests.log
TFFT_LIB=paper_2412_05824_b200/libtfft_tune.so python tools/tune_k1.py > $OUT/tune.log 2>&1
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > $OUT/bench2.json 2> $OUT/bench2.err
