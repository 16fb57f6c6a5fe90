# full -m gpu suite (verbose names) + the default bench line
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -rfE > gpurun_out/r2_full_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r2_full_tests.log
timeout 1200 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?"
tail -c 3500 gpurun_out/r2_bench.json; tail -3 gpurun_out/r2_bench.err
