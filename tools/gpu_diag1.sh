mkdir -p gpurun_out
timeout 600 python tools/roc_diag.py > gpurun_out/roc_diag.log 2>&1
head -30 gpurun_out/roc_diag.log
sed -i 's/timeout 900 ncu/timeout 300 ncu/' tools/gpu_prof.sh
bash tools/gpu_prof.sh "k5abft_fp32_4096 k5_kernel 2 1 --n 4096 --prec single --abft" "k5_fp32_4096 k5_kernel 1 1 --n 4096 --prec single" "k5abft_fp64_4096 k5_kernel 2 1 --n 4096 --prec double --abft" > /dev/null 2>&1
ls gpurun_out
