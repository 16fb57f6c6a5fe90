set -x
nproc; free -g; lscpu | head -20; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -c "import numpy; numpy.show_config()" 2>&1 | grep -i -A3 blas | head -20
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r2a_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/r2a_pytest.log
timeout 900 python scripts/run_configs.py cfg2 cfg3 cfg4 cfg5 > gpurun_out/r2a_configs.jsonl 2>&1; echo cfg rc=$?
cat gpurun_out/r2a_configs.jsonl
