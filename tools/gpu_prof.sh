#!/usr/bin/env bash
# ncu captures of the hot kernels, summarised to CSV on the box (.ncu-rep deleted)
OUT=gpurun_out
mkdir -p $OUT
summ() {
  ncu -i $OUT/$1.ncu-rep --page raw --csv > $OUT/$1.raw.csv 2>/dev/null
  ncu -i $OUT/$1.ncu-rep --page details --csv > $OUT/$1.details.csv 2>/dev/null
  ncu -i $OUT/$1.ncu-rep --page source --csv > $OUT/$1.source.csv 2>/dev/null
  gzip -f $OUT/$1.source.csv
  rm -f $OUT/$1.ncu-rep
}
prof() {  # tag, kernel regex, launches to skip, count, prof_one args
  tag=$1; kre=$2; skip=$3; cnt=$4; shift 4
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c $cnt -o $OUT/prof_$tag \
      python tools/prof_one.py "$@" --reps 3 > $OUT/prof_$tag.log 2>&1
  summ prof_$tag
}
for spec in "$@"; do
  eval prof $spec
done
ls -la $OUT | tail -30
