python scripts/host_copy_probe.py
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_api.py -q -m gpu -p no:cacheprovider -x > gpurun_out/r2_run5_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r2_run5_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -s -m gpu -p no:cacheprovider -k "cfg3_power_id" > gpurun_out/r2_run5_id.log 2>&1; echo id rc=$?
grep "cfg3 power_id" gpurun_out/r2_run5_id.log; tail -2 gpurun_out/r2_run5_id.log
timeout 600 python scripts/id_timeline.py cfg3 > gpurun_out/r2_id_cfg3_2lvl.txt 2>&1; head -14 gpurun_out/r2_id_cfg3_2lvl.txt
