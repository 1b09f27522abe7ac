# Multi-rank host logic of bench.py (strip plan, per-rank strip join, count
# exchange, max-over-ranks timing, e2e strip_join) on a ONE-GPU box: N ranks
# share cuda:0 and use gloo collectives (PBSM_BENCH_SHARED_GPU=1).  The ranks'
# kernels never wait on each other; the printed numbers are not measurements.
mkdir -p gpurun_out
for n in 2 4; do
  PBSM_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29500 + n)) bench.py --gpus $n --steps 3 --warmup 3 \
    --no-cpu-baseline > gpurun_out/multirank_$n.json 2> gpurun_out/multirank_$n.err
  echo "world $n rc=$?"; head -c 600 gpurun_out/multirank_$n.json; echo; tail -3 gpurun_out/multirank_$n.err
done
