#!/usr/bin/env bash
# the C2 sweep only (device-resident, no e2e / CPU / ABFT legs)
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-abft --sweep ${SWEEP:-13-20} > $OUT/bench_sweep.json 2> $OUT/bench_sweep.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_sweep.json').read().strip().splitlines()[-1])
for s in d['sweep']: print(s['n'], s['ms'], s['hbm_frac'])
PY
