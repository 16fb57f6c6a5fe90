# N > 1 bench code path of the DEFAULT workload (cfg4, strong scaling) on one GPU
# (gloo, all ranks on cuda:0): crash check only, never a measurement
for n in 2 8; do
SPB_BENCH_DRYRUN=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n \
  bench.py --gpus $n --steps 2 --warmup 3 --no-cpu > gpurun_out/r2g_dry_default_$n.json 2> gpurun_out/r2g_dry_default_$n.err
echo "default n=$n rc=$?"; tail -c 1200 gpurun_out/r2g_dry_default_$n.json; tail -n 3 gpurun_out/r2g_dry_default_$n.err
done
SPB_BENCH_DRYRUN=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29540 \
  bench.py --impl reference --gpus 8 --steps 2 --warmup 1 > gpurun_out/r2g_dry_ref8.json 2> gpurun_out/r2g_dry_ref8.err
echo "ref n=8 rc=$?"; tail -c 400 gpurun_out/r2g_dry_ref8.json
