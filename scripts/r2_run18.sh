timeout 600 python scripts/bj_probe.py 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_dense.py tests/test_gpu_kernels.py tests/test_gpu_twopass.py tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider > gpurun_out/r2_run18.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2_run18.log
