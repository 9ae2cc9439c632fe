# one gpurun call: full GPU test suite + compute-sanitizer over every kernel route
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rs -p no:cacheprovider > gpurun_out/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/tests.log
grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/tests.log | tail -15
bash tools/gpu_sanitize.sh
