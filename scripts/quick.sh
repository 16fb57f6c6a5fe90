#!/bin/bash
# quick GPU iteration: timeline of cfg2, short bench, optional gpu tests (QUICK_TESTS=1)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
export SPB_NO_BUILD=1
timeout 300 python scripts/timeline.py ${TL_CFG:-cfg2} 3 > gpurun_out/timeline.txt 2>&1
timeout 300 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_quick.log 2>&1
if [ -n "$QUICK_TESTS" ]; then
  timeout 600 python -m pytest tests -m gpu -q -x --timeout 120 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
fi
