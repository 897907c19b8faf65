# round 2, call F: Dot2 sign fix -- MLP parity tests; fused-kernel phase profile + ncu at k = 4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_f.txt; : > $S
timeout 1200 python -m pytest -q -rfs -k "mlp" tests/test_gpu_parity.py > gpurun_out/f_pytest_mlp.log 2>&1; echo pytest=$? >> $S
for k in 4 16; do
  SMA_MLP_PROF=500 timeout 300 python bench.py --config MLP --k $k --steps 1000 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/f_prof_k$k.log 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mlp_round_kernel -s 20 -c 1 -o gpurun_out/f_ncu_mlp_k4 python bench.py --config MLP --k 4 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/f_ncu.log 2>&1; echo ncu=$? >> $S
echo done >> $S
