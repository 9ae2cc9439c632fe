OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/tests.log; tail -2 $OUT/tests.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --sweep 8-8 > $OUT/bench_abft.json 2>&1
python -c "
import json
d=json.loads(open('$OUT/bench_abft.json').read().strip().splitlines()[-1])
for k,v in d['abft'].items(): print(k, v['plain_ms'], v['fused_ms'], v['overhead_pct'])
"
