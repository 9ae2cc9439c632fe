#!/usr/bin/env bash
# one gpurun call: K7 ring schedule sweep ("group_MB lag slots") over the two-pass sizes
OUT=gpurun_out
mkdir -p $OUT
: > $OUT/sched.log
for P in ${PRECS:-double single}; do
  TP_PREC=$P timeout 300 python tools/two_pass_ab.py | sed "s/^/default 0 0 /" >> $OUT/sched.log 2>&1
  for C in ${CONFIGS:-"16 1 4" "16 2 4" "16 2 5" "8 2 6" "8 3 6" "8 4 8" "12 2 5" "32 1 3"}; do
    set -- $C
    TFFT_K7_GROUP_MB=$1 TFFT_K7_LAG=$2 TFFT_K7_SLOTS=$3 TP_PREC=$P timeout 300 python tools/two_pass_ab.py | sed "s/^/$1 $2 $3 /" >> $OUT/sched.log 2>&1
  done
done
cat $OUT/sched.log
