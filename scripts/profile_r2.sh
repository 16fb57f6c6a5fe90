#!/bin/bash
# Round-2 profiles: launch list of the default (cfg4) bench step, --set full of
# the A pass (K2) and the gather, launch lists of one power_id call (cfg3,
# cfg5), the FP64 peaks.  Every ncu command follows the same command's plain
# run that exited 0.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
export SPB_NO_BUILD=1
mkdir -p gpurun_out
python scripts/fp64_peak.py > gpurun_out/r2_fp64_peak.json 2>&1; cat gpurun_out/r2_fp64_peak.json
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra"
timeout 600 $B > gpurun_out/r2p_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2_bench_launches_cfg4.csv $B > gpurun_out/r2p_ncu_launches.log 2>&1
echo "launch list rc=$?"
B1="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-extra"
timeout 600 $B1 > gpurun_out/r2p_plain1.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"skinny_tma|srht" -s 4 -c 2 \
  -o gpurun_out/r2_prof_cfg4 $B1 > gpurun_out/r2p_ncu_full.log 2>&1
echo "full rc=$?"
for c in cfg3 cfg5; do
  timeout 600 python scripts/id_call.py $c > gpurun_out/r2p_id_$c.log 2>&1 && \
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2_id_launches_$c.csv python scripts/id_call.py $c > gpurun_out/r2p_ncu_id_$c.log 2>&1
  echo "id $c rc=$?"; cat gpurun_out/r2p_id_$c.log
done
ls -la gpurun_out | head -30
