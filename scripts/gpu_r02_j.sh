# round 2, call J (barrier buffer size fixed): fused MLP round -- flag barrier, two-column z slice, dW1 register tile, z of b1/W2 staged
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_j.txt; : > $S
timeout 1200 python -m pytest -q -x -rfs -k "mlp" tests/test_gpu_parity.py > gpurun_out/j_pytest.log 2>&1; echo pytest=$? >> $S
for c in 0; do for k in 4 8 16 32; do
  SMA_MLP_COOP=$c SMA_MLP_PROF=500 timeout 300 python bench.py --config MLP --k $k --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/j_prof_c${c}_k$k.log 2>&1
  SMA_MLP_COOP=$c timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/j_bencj_c${c}_k$k.log 2>&1
done; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mlp_round_kernel -s 20 -c 1 -o gpurun_out/j_ncu_mlp_k4 python bench.py --config MLP --k 4 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/j_ncu.log 2>&1; echo ncu=$? >> $S
echo done >> $S
