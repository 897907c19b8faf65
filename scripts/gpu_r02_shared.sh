# round 2: the N > 1 code path of bench.py end to end with all ranks time-sharing cuda:0
# (SMA_BENCH_SHARED_GPU=1: a path test, not a measurement), after the round-2 bench changes
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_shared2.txt; : > $S
for n in 2 4; do
  SMA_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 30 --warmup 3 > gpurun_out/sh2_n$n.log 2>&1; echo n$n=$? >> $S
  SMA_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $n --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --hier > gpurun_out/sh2_hier_n$n.log 2>&1; echo hier_n$n=$? >> $S
  SMA_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $n --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --config MLP --rounds-per-call 30 > gpurun_out/sh2_mlp_n$n.log 2>&1; echo mlp_n$n=$? >> $S
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --impl reference --gpus 2 --steps 3 --warmup 1 > gpurun_out/sh2_ref_n2.log 2>&1; echo ref_n2=$? >> $S
echo done >> $S
