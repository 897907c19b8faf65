# round 2, call G: fused MLP round with one grid barrier + TMA-staged blocks -- MLP tests, phase profile, bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_g.txt; : > $S
timeout 1200 python -m pytest -q -x -rfs -k "mlp" tests/test_gpu_parity.py > gpurun_out/g_pytest_mlp.log 2>&1; echo pytest=$? >> $S
for k in 4 8 16 32; do
  SMA_MLP_PROF=500 timeout 300 python bench.py --config MLP --k $k --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/g_prof_k$k.log 2>&1
  timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/g_bench_k$k.log 2>&1
done
echo done >> $S
