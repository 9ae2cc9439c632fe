# one gpurun call: full GPU tests, smoke, bench (+ reference arm), launch list of one
# bench step, ncu captures of the dominant kernels, sanitizers; everything under gpurun_out/
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rs -p no:cacheprovider > $OUT/tests.log 2>&1; echo "tests rc=$?" >> $OUT/tests.log
tail -3 $OUT/tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
tail -c 400 $OUT/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-abft > /dev/null 2>&1
sed -i 's/timeout 900 ncu/timeout 300 ncu/' tools/gpu_prof.sh
bash tools/gpu_prof.sh "k7_fp64_n1m k7_kernel 1 1 --n 1048576 --prec double" "k7_fp64_n65536 k7_kernel 1 1 --n 65536 --prec double" \
  "k5_fp64_n4096 k5_kernel 1 1 --n 4096 --prec double" "k5abft_fp32_n4096 k5_abft2 1 1 --n 4096 --prec single --abft" \
  "k5abft_fp64_n4096 k5_kernel 2 1 --n 4096 --prec double --abft" "k4_fp32_n65536 k4_kernel 1 1 --n 65536 --prec single" \
  "stage_fp64_n8m col_kernel 1 1 --n 8388608 --prec double" "winfin_fp32_n4096 k5_window 1 1 --n 4096 --prec single --abft" > /dev/null 2>&1
bash tools/gpu_sanitize.sh > /dev/null 2>&1
cat $OUT/sanitizer/summary.txt
