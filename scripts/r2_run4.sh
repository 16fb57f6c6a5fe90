timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_ingest.py -q -s -m gpu -p no:cacheprovider > gpurun_out/r2_run4_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/r2_run4_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -s -m gpu -p no:cacheprovider -k "cfg3_power_id" > gpurun_out/r2_run4_id.log 2>&1; echo id rc=$?
grep "cfg3 power_id" gpurun_out/r2_run4_id.log; tail -2 gpurun_out/r2_run4_id.log
timeout 1200 python bench.py > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err; echo bench rc=$?
tail -c 4000 gpurun_out/r2_bench_default.json; tail -5 gpurun_out/r2_bench_default.err
