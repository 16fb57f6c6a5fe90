timeout 1200 python scripts/bj_probe.py 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_dense.py -q -m gpu -p no:cacheprovider -x > gpurun_out/r2_run10_dense.log 2>&1; echo "dense rc=$?"; tail -3 gpurun_out/r2_run10_dense.log
