# GPU parity run: the full-size + API tests first (verbose, -s for the printed
# per-quantity errors), then the whole -m gpu suite
timeout 1500 python -m pytest tests/test_gpu_api.py tests/test_gpu_fullsize.py -q -s -m gpu -p no:cacheprovider > gpurun_out/r2_new_tests.log 2>&1; echo new rc=$?
tail -5 gpurun_out/r2_new_tests.log
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider --deselect tests/test_gpu_fullsize.py > gpurun_out/r2_all_tests.log 2>&1; echo all rc=$?
tail -3 gpurun_out/r2_all_tests.log
