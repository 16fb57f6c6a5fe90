timeout 900 python scripts/id_call.py cfg5 2>&1 | tail -2
timeout 600 python scripts/id_timeline.py cfg5 2>/dev/null | head -14
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_api.py tests/test_gpu_sharded.py -q -s -m gpu -p no:cacheprovider -k "cfg5 or id or sharded" > gpurun_out/r2_run16.log 2>&1; echo "tests rc=$?"; grep -E "cfg3 power_id|cfg5|passed|failed" gpurun_out/r2_run16.log | tail -8
