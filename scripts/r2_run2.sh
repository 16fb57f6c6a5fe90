timeout 1200 python -m pytest tests/test_gpu_dense.py tests/test_gpu_api.py -q -s -m gpu -p no:cacheprovider -x > gpurun_out/r2_dense.log 2>&1; echo dense rc=$?
tail -3 gpurun_out/r2_dense.log
timeout 600 python scripts/id_timeline.py cfg3 > gpurun_out/r2_id_cfg3.txt 2>&1
timeout 600 python scripts/id_timeline.py cfg5 > gpurun_out/r2_id_cfg5.txt 2>&1
cat gpurun_out/r2_id_cfg3.txt gpurun_out/r2_id_cfg5.txt | head -70
