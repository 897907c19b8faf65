# round 2, call S: fused MLP kernel -- x-norm fix; group-2 size sweep (SMA_MLP_ZWARPS 0/2/4), per-call and multi-round
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_s.txt; : > $S
timeout 1200 python -m pytest -q -x -rfs -k "mlp or learner_steps" tests/test_gpu_parity.py > gpurun_out/s_pytest.log 2>&1; echo pytest=$? >> $S
for zw in 0 2 4; do for k in 4 8 16; do
  SMA_MLP_ZWARPS=$zw timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/s_b1_z${zw}_k$k.log 2>&1
  SMA_MLP_ZWARPS=$zw timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --rounds-per-call 3000 --no-cpu-baseline --no-e2e > gpurun_out/s_bM_z${zw}_k$k.log 2>&1
done; done
echo done >> $S
