#!/usr/bin/env bash
# ncu launch list of one C5 protected call (FP32 N=2^16, 1 GiB, T=8)
OUT=gpurun_out; mkdir -p $OUT
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/c5_launches.csv python tools/prof_one.py --n 65536 --prec single --abft --reps 2 > /dev/null 2>&1
python - <<'PY'
import csv
r = list(csv.reader(l for l in open('gpurun_out/c5_launches.csv') if not l.startswith('==')))
h = r[0]
for x in r[1:]:
    print(x[h.index('Kernel Name')][:45], x[h.index('Metric Name')], x[h.index('Metric Value')])
PY
