#!/bin/bash
# Round-2 (final) profile pass, run on the GPU box through gpurun:
#   gpurun --timeout 3000 -- 'bash scripts/profile_r2.sh'
# Every profiled command first runs plain (must exit 0); numbers printed under
# ncu are never bench values.  Outputs land in gpurun_out/ and are summarised
# into profiles/ here (scripts/launch_shares.py, scripts/ncu_summary.py).
set -u
O=gpurun_out
mkdir -p $O
NCU_LIST="ncu --metrics gpu__time_duration.sum --clock-control none --csv"
B4="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra"
B2="python bench.py --config cfg2 --steps 5 --warmup 3 --no-e2e --no-cpu --no-extra"
B3="python bench.py --config cfg3 --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra"
$B4 > $O/r2f_plain_cfg4.json 2> $O/r2f_plain_cfg4.err || { echo "plain cfg4 failed"; exit 1; }
$NCU_LIST --log-file $O/r2f_launches_cfg4.csv $B4 > $O/r2f_ncu_cfg4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'skinny_tma|srht' -s 4 -c 2 -f -o $O/r2f_prof_cfg4 \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-extra > $O/r2f_ncu_full_cfg4.log 2>&1
$B2 > $O/r2f_plain_cfg2.json 2> $O/r2f_plain_cfg2.err && \
  $NCU_LIST --log-file $O/r2f_launches_cfg2.csv $B2 > $O/r2f_ncu_cfg2.log 2>&1
$B3 > $O/r2f_plain_cfg3.json 2> $O/r2f_plain_cfg3.err && \
  $NCU_LIST --log-file $O/r2f_launches_cfg3.csv $B3 > $O/r2f_ncu_cfg3.log 2>&1
for c in cfg3 cfg5; do
  python scripts/id_call.py $c > $O/r2f_id_plain_$c.log 2>&1 && \
    $NCU_LIST --log-file $O/r2f_id_launches_$c.csv python scripts/id_call.py $c > $O/r2f_id_ncu_$c.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:'jacobi_blk' -s 2 -c 1 -f -o $O/r2f_prof_jblk \
    python scripts/id_call.py cfg3 > $O/r2f_ncu_full_jblk.log 2>&1
ls -la $O | tail -30
