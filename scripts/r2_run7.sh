timeout 600 python -m pytest tests/test_gpu_sharded.py -q -s -m gpu -p no:cacheprovider > gpurun_out/r2_run7_tests.log 2>&1; echo tests rc=$?
grep -E "passed|failed|^E " gpurun_out/r2_run7_tests.log | head -12
bash scripts/run_reftests.sh
