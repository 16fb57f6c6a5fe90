#!/bin/bash
# Diagnostic: rebuild with the Jacobi sweep trace on the box and run one
# power_svd per config (sweeps per Rayleigh-Ritz core printed by the kernel).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
SPB_NVCC_EXTRA="-DSPB_JACOBI_TRACE" python -c "from paper_2105_01271_b200.build import build; build(force=True)" > gpurun_out/jt_build.log 2>&1
for c in ${CFGS:-cfg2 cfg3}; do
  SPB_NO_BUILD=1 timeout 300 python scripts/timeline.py $c 1 > gpurun_out/jt_$c.txt 2>&1
done
