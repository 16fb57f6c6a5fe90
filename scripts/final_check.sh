set -u
O=gpurun_out
NCU_LIST="ncu --metrics gpu__time_duration.sum --clock-control none --csv"
python -m pytest tests -m gpu -x -q > $O/s4_gputest3.log 2>&1; tail -2 $O/s4_gputest3.log
for c in cfg3 cfg5; do
  python scripts/id_call.py $c > $O/r2f_id_plain_$c.log 2>&1 && \
    $NCU_LIST --log-file $O/r2f_id_launches_$c.csv python scripts/id_call.py $c > $O/r2f_id_ncu_$c.log 2>&1
done
python bench.py > $O/s4_bench5.json 2> $O/s4_bench5.err; tail -2 $O/s4_bench5.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/s4_bench5_ref.json 2>&1
