#!/bin/bash
# Profiles for profiles/: the launch list of a short bench run (ncu
# gpu__time_duration, cold-cache serialised) and one --set full capture of
# each top kernel.  One GPU; every ncu run follows a plain run that exited 0.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
export SPB_NO_BUILD=1
mkdir -p gpurun_out
ARGS="--steps 5 --warmup 3 --no-e2e --no-cpu"
timeout 300 python bench.py $ARGS > gpurun_out/plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launches.log 2>&1
A1="--steps 1 --warmup 0 --no-e2e --no-cpu"
timeout 300 python bench.py $A1 > gpurun_out/plain1.log 2>&1 || exit 1
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"${KREGEX:-skinny_tma|tsqr_leaf|jacobi32|srht|finish_core|stencil|gram_rows|finish_rows|dgemm|tsqr_apply|ddgram}" \
  -s ${SKIP:-40} -c ${COUNT:-12} -o gpurun_out/prof_full python bench.py $A1 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out/
