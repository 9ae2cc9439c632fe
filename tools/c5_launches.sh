OUT=gpurun_out; mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/c5_launches.csv python tools/prof_one.py --n 65536 --prec single --abft --bytes 536870912 --reps 2 > /dev/null 2>&1
cat $OUT/c5_launches.csv | grep -v "^==" | awk -F'","' '{print $5, $(NF)}' | tail -30
