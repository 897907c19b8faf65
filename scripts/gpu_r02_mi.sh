# round 2, call MI: fused MLP kernel, b = 16, classes = 10 and in_dim = 784 as compile-time constants -- multi-round rates k = 4 / 8 / 16, profile k = 4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_mi.txt; : > $S
for k in 4 8 16 32; do
  timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --rounds-per-call 3000 --no-cpu-baseline --no-e2e > gpurun_out/mi_k$k.log 2>&1; echo k$k=$? >> $S
done
SMA_MLP_PROF=3 timeout 300 python bench.py --config MLP --k 4 --steps 1000 --warmup 20 --rounds-per-call 1000 --no-cpu-baseline --no-e2e > gpurun_out/mi_prof.log 2>&1
echo done >> $S
timeout 1500 python -m pytest -q -x -rfs tests/test_gpu_parity.py -k "mlp" > gpurun_out/mi_pytest.log 2>&1; echo pytest=$? >> $S
