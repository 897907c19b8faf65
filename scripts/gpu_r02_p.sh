# round 2, call P: multi-round fused MLP kernel with the z slice on 2 warps beside phase 1, G only in the last round
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_p.txt; : > $S
timeout 1200 python -m pytest -q -x -rfs -k "mlp or learner_steps" tests/test_gpu_parity.py > gpurun_out/p_pytest.log 2>&1; echo pytest=$? >> $S
for k in 4 8 16 32; do
  timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/p_bench1_k$k.log 2>&1
  timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --rounds-per-call 3000 --no-cpu-baseline --no-e2e > gpurun_out/p_benchM_k$k.log 2>&1
done
SMA_MLP_PROF=3 timeout 300 python bench.py --config MLP --k 4 --steps 1000 --warmup 20 --rounds-per-call 1000 --no-cpu-baseline --no-e2e > gpurun_out/p_prof_k4.log 2>&1
echo done >> $S
