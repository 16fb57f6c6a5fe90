#!/bin/bash
# Diagnostic: rebuild with the clock64 phase timers on the box and run one
# power_svd per config (phase cycle counts printed by the instrumented kernels).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
SPB_NVCC_EXTRA="-DSPB_PHASE_TRACE" python -c "from paper_2105_01271_b200.build import build; build(force=True)" > gpurun_out/pt_build.log 2>&1
for c in ${CFGS:-cfg2}; do
  SPB_NO_BUILD=1 timeout 300 python scripts/timeline.py $c 1 > gpurun_out/pt_$c.txt 2>&1
done
