#!/bin/bash
# ncu --set full captures of the top kernels (one GPU, after a plain run exited 0)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
export SPB_NO_BUILD=1
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 || exit 1
for k in ${KERNELS:-skinny_atz tsqr_leaf jacobi chol_inv dgemm}; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/prof_$k python bench.py $ARGS > gpurun_out/ncu_$k.log 2>&1
done
ls -la gpurun_out/
