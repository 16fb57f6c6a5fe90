timeout 1500 python -m pytest tests/test_gpu_dense.py tests/test_gpu_api.py tests/test_gpu_fullsize.py -q -s -m gpu -p no:cacheprovider > gpurun_out/r2_run3_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/r2_run3_tests.log
timeout 600 python scripts/id_timeline.py cfg3 > gpurun_out/r2_id_cfg3_exact.txt 2>&1; head -12 gpurun_out/r2_id_cfg3_exact.txt
timeout 900 python bench.py > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err; echo bench rc=$?
tail -c 3000 gpurun_out/r2_bench_default.json; tail -5 gpurun_out/r2_bench_default.err
