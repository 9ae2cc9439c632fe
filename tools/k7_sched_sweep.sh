#!/usr/bin/env bash
# one gpurun call: two-pass ring group-size sweep (TFFT_K4_GROUP_MB) over the two-pass sizes
OUT=gpurun_out
mkdir -p $OUT
: > $OUT/sched.log
for P in ${PRECS:-double single}; do
  TP_PREC=$P timeout 300 python tools/two_pass_ab.py | sed "s/^/default 0 0 /" >> $OUT/sched.log 2>&1
  for M in ${GROUPS_MB:-12 16 20 24 28 40}; do
    TFFT_K4_GROUP_MB=$M TP_PREC=$P timeout 300 python tools/two_pass_ab.py | sed "s/^/$M 1 3 /" >> $OUT/sched.log 2>&1
  done
done
python tools/sched_table.py
