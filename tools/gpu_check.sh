#!/usr/bin/env bash
# one gpurun call: GPU tests (optionally a -k filter), smoke, short bench; logs under gpurun_out/
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
K=${K:-}
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -x --timeout 600 ${K:+-k "$K"} -rs > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/tests.log
tail -15 $OUT/tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
tail -2 $OUT/smoke.log
if [ -n "$BENCH" ]; then
  timeout 600 python bench.py --steps 5 --warmup 3 $BENCH > $OUT/bench.json 2> $OUT/bench.err
  tail -c 1500 $OUT/bench.json
fi
