mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_prot32.csv python tools/prof_one.py --n 4096 --prec single --abft --reps 2 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_prot64.csv python tools/prof_one.py --n 4096 --prec double --abft --reps 2 > /dev/null 2>&1
bash tools/gpu_prof.sh "k5abft_fp32_4096 k5_kernel 2 1 --n 4096 --prec single --abft" "k5_fp32_4096 k5_kernel 1 1 --n 4096 --prec single" > /dev/null 2>&1
ls gpurun_out
