# launch lists (ncu gpu__time_duration) of protected calls: args = "n prec" pairs
mkdir -p gpurun_out
while [ $# -gt 1 ]; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${1}_${2}.csv \
      python tools/prof_one.py --n $1 --prec $2 --abft --reps 2 > /dev/null 2>&1
  python tools/launch_table.py gpurun_out/launches_${1}_${2}.csv
  shift 2
done
