timeout 900 python bench.py --config cfg2 --no-e2e --no-cpu --steps 30 > gpurun_out/r2_b9.json 2> gpurun_out/r2_b9.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2_b9.json').read().strip().splitlines()[-1])
print('cfg2', d['ms_per_step'], d['value'], d['clocks']); print(json.dumps({k: (v['ms'], v.get('power_id')) for k, v in d['other_configs'].items()}))"
timeout 600 python scripts/timeline.py cfg2 3 > gpurun_out/r2_timeline_cfg2.txt 2>&1; head -30 gpurun_out/r2_timeline_cfg2.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -s -m gpu -p no:cacheprovider -k "power_id" > gpurun_out/r2_b9_id.log 2>&1; grep "cfg3 power_id" gpurun_out/r2_b9_id.log; tail -1 gpurun_out/r2_b9_id.log
