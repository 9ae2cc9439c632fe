#!/usr/bin/env bash
# one gpurun call: two-pass timings (tools/two_pass_ab.py) for the production lib
# and each experiment lib in LIBS (space-separated tags: paper_2412_05824_b200/libtfft_<tag>.so),
# optional DRAM bytes of the K7 launch at the sizes in DRAM_N, then the GPU tests (K filter; NOTESTS=1 skips)
OUT=gpurun_out
mkdir -p $OUT
for P in ${PRECS:-double single}; do
  TP_PREC=$P timeout 300 python tools/two_pass_ab.py > $OUT/ab_prod_$P.log 2>&1
  for L in $LIBS; do
    TFFT_LIB=paper_2412_05824_b200/libtfft_$L.so TP_PREC=$P timeout 300 python tools/two_pass_ab.py > $OUT/ab_${L}_$P.log 2>&1
  done
done
tail -n 20 $OUT/ab_*.log
for N in $DRAM_N; do
  for L in prod $LIBS; do
    LIBV=""; [ "$L" != prod ] && LIBV=paper_2412_05824_b200/libtfft_$L.so
    TFFT_LIB=$LIBV timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k7_kernel -c 1 \
      python tools/prof_one.py --n $N --prec double --reps 1 > $OUT/dram_${L}_$N.log 2>&1
    grep -E 'dram__bytes|gpu__time' $OUT/dram_${L}_$N.log | sed "s/^/$L $N /"
  done
done
if [ -z "$NOTESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 ${K:+-k "$K"} > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/tests.log
  tail -4 $OUT/tests.log
fi
