# N > 1 bench code path on one GPU (gloo, all ranks on cuda:0): crash check only
for n in 2 4; do
SPB_BENCH_DRYRUN=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n \
  bench.py --gpus $n --steps 3 --warmup 3 --config cfg2 --no-cpu > gpurun_out/r2_dry_$n.json 2> gpurun_out/r2_dry_$n.err
echo "n=$n rc=$?"; tail -c 1500 gpurun_out/r2_dry_$n.json; tail -3 gpurun_out/r2_dry_$n.err
done
SPB_BENCH_DRYRUN=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29520 \
  bench.py --gpus 2 --steps 2 --warmup 3 --config cfg3 --no-cpu --no-e2e > gpurun_out/r2_dry_cfg3.json 2> gpurun_out/r2_dry_cfg3.err
echo "cfg3 n=2 rc=$?"; tail -c 800 gpurun_out/r2_dry_cfg3.json; tail -3 gpurun_out/r2_dry_cfg3.err
SPB_BENCH_DRYRUN=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/r2_dry_ref.json 2> gpurun_out/r2_dry_ref.err
echo "ref n=2 rc=$?"; tail -c 600 gpurun_out/r2_dry_ref.json
