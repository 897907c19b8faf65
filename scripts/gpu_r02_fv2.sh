# round 2, call FV2: final validation (after the compile-time in_dim in the MLP kernel) -- smoke, every GPU test, the default bench line, the other configs, the
# reference arm, C1 convergence, the C4 launch list, and bench.py's N > 1 path with 2 ranks time-sharing the GPU
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_fv2.txt; : > $S
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fv2_smoke.log 2>&1; echo smoke=$? >> $S
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rfs > gpurun_out/fv2_pytest_gpu.log 2>&1; echo pytest=$? >> $S
timeout 600 python bench.py > gpurun_out/fv2_bench.log 2>&1; echo bench=$? >> $S
: > gpurun_out/fv2_other.jsonl
for c in C2 C3 C5; do timeout 300 python bench.py --config $c --steps 2000 --warmup 50 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' >> gpurun_out/fv2_other.jsonl; done
for rpc in 1 1000; do timeout 300 python bench.py --config C1 --steps 3000 --warmup 50 --rounds-per-call $rpc --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' >> gpurun_out/fv2_other.jsonl; done
for k in 4 8 16 32; do timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --rounds-per-call 3000 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' >> gpurun_out/fv2_other.jsonl; done
echo other=$? >> $S
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fv2_ref.log 2>&1; echo ref=$? >> $S
timeout 300 python scripts/c1_convergence.py > gpurun_out/fv2_c1_convergence.jsonl 2> gpurun_out/fv2_c1_convergence.err; echo conv=$? >> $S
SMA_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 30 --warmup 3 > gpurun_out/fv2_shared_n2.log 2>&1; echo shared_n2=$? >> $S
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fv2_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fv2_ncu.log 2>&1; echo ncu=$? >> $S
echo done >> $S
