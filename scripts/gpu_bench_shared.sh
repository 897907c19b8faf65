cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for n in 2 4; do
  SMA_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench_shared_n$n.log 2>&1; echo n$n=$? >> gpurun_out/status_shared.txt
  SMA_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $n --steps 30 --warmup 3 --no-cpu-baseline --hier > gpurun_out/bench_shared_hier_n$n.log 2>&1; echo hier_n$n=$? >> gpurun_out/status_shared.txt
  SMA_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $n --steps 30 --warmup 3 --no-cpu-baseline --config MLP > gpurun_out/bench_shared_mlp_n$n.log 2>&1; echo mlp_n$n=$? >> gpurun_out/status_shared.txt
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --impl reference --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_ref_n2.log 2>&1; echo ref_n2=$? >> gpurun_out/status_shared.txt
echo done >> gpurun_out/status_shared.txt
