#!/bin/bash
# Round-2 (last session) profile pass on the GPU box:  gpurun --timeout 2400 -- 'bash scripts/profile_r2g.sh'
# Every profiled command first runs plain (must exit 0); numbers printed under ncu are never bench values.
set -u
O=gpurun_out
mkdir -p $O
NCU_LIST="ncu --metrics gpu__time_duration.sum --clock-control none --csv"
B4="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra"
B5="python bench.py --config cfg5 --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra"
/usr/bin/time -v python bench.py > $O/r2g_plain_default.json 2> $O/r2g_plain_default.err; echo "default bench rc=$?"; grep "Elapsed" $O/r2g_plain_default.err
$B4 > $O/r2g_plain_cfg4.json 2> $O/r2g_plain_cfg4.err || { echo "plain cfg4 failed"; exit 1; }
$NCU_LIST --log-file $O/r2g_launches_cfg4.csv $B4 > $O/r2g_ncu_cfg4.log 2>&1
$B5 > $O/r2g_plain_cfg5.json 2> $O/r2g_plain_cfg5.err && \
  $NCU_LIST --log-file $O/r2g_launches_cfg5.csv $B5 > $O/r2g_ncu_cfg5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'skinny_tma' -s 4 -c 1 -f -o $O/r2g_prof_k2 \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-extra > $O/r2g_ncu_full_k2.log 2>&1
ls -la $O | grep r2g
