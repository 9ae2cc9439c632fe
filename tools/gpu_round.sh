#!/usr/bin/env bash
# one gpurun call: bench + launch list + ncu captures of the hot kernels.
# .ncu-rep files are summarised to CSV on the box and deleted (gpurun copies
# back at most 64 MiB).
OUT=gpurun_out
mkdir -p $OUT
python bench.py --steps 5 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-abft > /dev/null 2>&1
summ() {  # $1 = report base name
  ncu -i $OUT/$1.ncu-rep --page raw --csv > $OUT/$1.raw.csv 2>/dev/null
  ncu -i $OUT/$1.ncu-rep --page details --csv > $OUT/$1.details.csv 2>/dev/null
  ncu -i $OUT/$1.ncu-rep --page source --csv > $OUT/$1.source.csv 2>/dev/null
  gzip -f $OUT/$1.source.csv
  rm -f $OUT/$1.ncu-rep
}
prof() {  # $1 = tag, rest = prof_one args
  tag=$1; shift
  timeout 900 ncu --set full --clock-control none --import-source on -s 2 -c 1 -o $OUT/prof_$tag \
      python tools/prof_one.py "$@" --reps 3 > $OUT/prof_$tag.log 2>&1
  summ prof_$tag
}
prof k1_fp64_n4096 --n 4096 --prec double
prof k1_fp32_n1024 --n 1024 --prec single
prof k1_fp64_n256 --n 256 --prec double
prof k3_fp64_n65536 --n 65536 --prec double
prof k3_fp64_n1m --n 1048576 --prec double
prof k1abft_fp32_n4096 --n 4096 --prec single --abft
ls -la $OUT
du -sh $OUT
