mkdir -p gpurun_out
bash tools/gpu_prof.sh "k5abft_fp32_4096 k5_kernel 2 1 --n 4096 --prec single --abft" "k5_fp32_4096 k5_kernel 1 1 --n 4096 --prec single" "k5abft_fp64_4096 k5_kernel 2 1 --n 4096 --prec double --abft" > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_prot.csv python tools/prof_one.py --n 4096 --prec single --abft --reps 2 > /dev/null 2>&1
ls -la gpurun_out
