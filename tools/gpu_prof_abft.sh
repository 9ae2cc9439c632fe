bash tools/gpu_prof.sh "k5abft_fp32_n4096 k5_kernel 1 1 --n 4096 --prec single --abft" "k5_fp32_n4096 k5_kernel 1 1 --n 4096 --prec single"
