mkdir -p gpurun_out
F="tests/refsuite/test_acceptance.py::test_criterion_3_roc_protocol tests/refsuite/test_fault.py::test_roc_campaign_rates tests/test_gpu_scale.py::test_one_fault_per_window tests/test_gpu_scale.py::test_roc_protocol_2000_runs tests/test_gpu_scale.py::test_criterion4_protocol tests/test_gpu_shard_mp.py tests/test_gpu_scale.py::test_scale_campaign_decisions"
TFFT_NO_K5_ABFT=1 timeout 900 python -m pytest $F -q --timeout 600 -x -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/iso_nok5.log
timeout 900 python -m pytest $F -q --timeout 600 -p no:cacheprovider 2>&1 | grep -E "passed|failed|^FAILED" > gpurun_out/iso_k5.log
ABFT_AB_LOGN=9,10,11,12,13 timeout 600 python tools/abft_ab.py > gpurun_out/abft_ab.log 2>&1
TFFT_NO_K5_ABFT=1 ABFT_AB_LOGN=9,10,11,12 timeout 600 python tools/abft_ab.py > gpurun_out/abft_ab_nok5.log 2>&1
cat gpurun_out/iso_nok5.log gpurun_out/iso_k5.log gpurun_out/abft_ab.log gpurun_out/abft_ab_nok5.log
