#!/usr/bin/env bash
# compute-sanitizer over every kernel route at small shapes (tools/sanitize_cases.py)
OUT=gpurun_out/sanitizer
mkdir -p $OUT
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_cases.py > $OUT/$tool.log 2>&1
  echo "$tool rc=$?" | tee -a $OUT/summary.txt
  tail -5 $OUT/$tool.log
done
