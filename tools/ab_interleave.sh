#!/usr/bin/env bash
# one gpurun call: interleaved two-pass timings, production lib vs libtfft_<tag>.so for each tag in LIBS, ROUNDS times
OUT=gpurun_out
mkdir -p $OUT
: > $OUT/abi.log
for i in $(seq ${ROUNDS:-2}); do
  for P in ${PRECS:-double single}; do
    TP_PREC=$P timeout 300 python tools/two_pass_ab.py | sed "s/^/prod $i /" >> $OUT/abi.log 2>&1
    for L in $LIBS; do
      TFFT_LIB=paper_2412_05824_b200/libtfft_$L.so TP_PREC=$P timeout 300 python tools/two_pass_ab.py | sed "s/^/$L $i /" >> $OUT/abi.log 2>&1
    done
  done
done
python tools/abi_table.py
