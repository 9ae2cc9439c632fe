OUT=gpurun_out; mkdir -p $OUT
TFFT_LIB=paper_2412_05824_b200/libtfft_tune.so timeout 1200 python tools/tune_k1.py > $OUT/tune.log 2>&1
tail -40 $OUT/tune.log
