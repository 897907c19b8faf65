# round 2, call K: fused MLP round -- split-phase flags (PL per learner, ZD before the first replica store), padded rows, z slice after the partial logits
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_k.txt; : > $S
timeout 1200 python -m pytest -q -x -rfs -k "mlp" tests/test_gpu_parity.py > gpurun_out/k_pytest.log 2>&1; echo pytest=$? >> $S
for k in 4 8 16 32; do
  SMA_MLP_PROF=500 timeout 300 python bench.py --config MLP --k $k --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/k_prof_k$k.log 2>&1
  timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/k_bench_k$k.log 2>&1
done
echo done >> $S
