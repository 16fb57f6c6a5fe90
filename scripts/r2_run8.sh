timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_api.py tests/test_gpu_parity.py tests/test_gpu_twopass.py -q -s -m gpu -p no:cacheprovider > gpurun_out/r2_run8_tests.log 2>&1; echo tests rc=$?
grep -E "passed|failed|^E  |sharded ID" gpurun_out/r2_run8_tests.log | head -12
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -s -m gpu -p no:cacheprovider -k "power_id or cfg5" > gpurun_out/r2_run8_id.log 2>&1; echo id rc=$?
grep -E "cfg3 power_id|cfg5|passed|failed" gpurun_out/r2_run8_id.log | head
bash scripts/run_reftests.sh
timeout 600 python scripts/id_timeline.py cfg5 > gpurun_out/r2_id_cfg5_exact.txt 2>&1; head -12 gpurun_out/r2_id_cfg5_exact.txt
