timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_ingest.py tests/test_gpu_api.py -q -s -m gpu -p no:cacheprovider > gpurun_out/r2_run6_tests.log 2>&1; echo tests rc=$?
grep "sharded ID\|passed\|failed" gpurun_out/r2_run6_tests.log | tail -8
timeout 900 python bench.py --config cfg2 --no-e2e --no-cpu --steps 20 > gpurun_out/r2_bench_cfg2.json 2> gpurun_out/r2_bench_cfg2.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_cfg2.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step']); print(json.dumps(d['other_configs'].get('cfg2', {}), indent=0)[:200]);
print(json.dumps({k: v.get('power_id') for k, v in d['other_configs'].items()}))"
tail -3 gpurun_out/r2_bench_cfg2.err
