cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/b2.txt
timeout 900 python bench.py > gpurun_out/b2_C4.log 2>&1; echo "C4 rc=$?" >> gpurun_out/b2.txt
for c in C1 MLP C2 C3 C5; do timeout 600 python bench.py --config $c --steps 3000 --no-cpu-baseline --no-e2e > gpurun_out/b2_$c.log 2>&1; echo "$c rc=$?" >> gpurun_out/b2.txt; done
timeout 600 python bench.py --force-collective --steps 300 --no-cpu-baseline --no-e2e > gpurun_out/b2_coll.log 2>&1; echo "coll rc=$?" >> gpurun_out/b2.txt
timeout 600 python bench.py --tau 4 --steps 300 --no-cpu-baseline --no-e2e > gpurun_out/b2_tau.log 2>&1; echo "tau rc=$?" >> gpurun_out/b2.txt
SMA_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/b2_shared2.log 2>&1; echo "shared2 rc=$?" >> gpurun_out/b2.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 500 -k "timing or kernel_time" > gpurun_out/b2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/b2.txt
