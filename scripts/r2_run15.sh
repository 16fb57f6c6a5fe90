timeout 600 python scripts/bj_timeline.py 5000 4096 2>/dev/null | head -8
timeout 600 python scripts/bj_probe.py 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_dense.py -q -m gpu -p no:cacheprovider -x > gpurun_out/r2_run15_dense.log 2>&1; echo "dense rc=$?"; tail -2 gpurun_out/r2_run15_dense.log
