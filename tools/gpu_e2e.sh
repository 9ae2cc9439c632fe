OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/tests.log; tail -2 $OUT/tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-abft > $OUT/bench_e2e.json 2>&1
python -c "
import json
d=json.loads(open('$OUT/bench_e2e.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e'], d.get('c1'))
"
