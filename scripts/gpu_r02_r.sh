# round 2, call R: fused MLP kernel -- group 2 (2 warps) owns the next round's rows/norms, the z slice, the ZD wait
# and the z-block prefetch; small phase-2 items on the threads without a dW1 item; z rows preloaded in dW1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_r.txt; : > $S
timeout 1200 python -m pytest -q -x -rfs -k "mlp or learner_steps" tests/test_gpu_parity.py > gpurun_out/r_pytest.log 2>&1; echo pytest=$? >> $S
for k in 4 8 16 32; do
  timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/r_bench1_k$k.log 2>&1
  timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --rounds-per-call 3000 --no-cpu-baseline --no-e2e > gpurun_out/r_benchM_k$k.log 2>&1
done
for k in 4 16; do
SMA_MLP_PROF=3 timeout 300 python bench.py --config MLP --k $k --steps 1000 --warmup 20 --rounds-per-call 1000 --no-cpu-baseline --no-e2e > gpurun_out/r_prof_k$k.log 2>&1
done
echo done >> $S
