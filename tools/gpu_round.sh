#!/usr/bin/env bash
# one gpurun call: bench + launch list + ncu captures of the hot kernels
set -x
OUT=gpurun_out
python bench.py --steps 5 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-abft > /dev/null 2>&1
for cfg in "--n 4096 --prec double" "--n 1024 --prec single" "--n 65536 --prec double" "--n 1048576 --prec double"; do
  tag=$(echo $cfg | tr -d ' -' )
  timeout 600 ncu --set full --clock-control none --import-source on -s 2 -c 2 -o $OUT/prof_$tag \
      python tools/prof_one.py $cfg --reps 2 > $OUT/prof_$tag.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_kernel -s 1 -c 1 -o $OUT/prof_abft_n4096_fp32 \
    python tools/prof_one.py --n 4096 --prec single --abft --reps 2 > $OUT/prof_abft.log 2>&1
ls -la $OUT
