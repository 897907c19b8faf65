# round 2, call RP: fused MLP kernel, flag polls with relaxed loads + one acquire fence
# (SMA_MLP_RELAXPOLL=1 vs 0), multi-round rates at k = 4 / 8 / 16, phase profile, the MLP parity tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_rp.txt; : > $S
for rel in 1 0; do
  for k in 4 8 16; do
    SMA_MLP_RELAXPOLL=$rel timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --rounds-per-call 3000 --no-cpu-baseline --no-e2e > gpurun_out/rp_rel${rel}_k$k.log 2>&1; echo rel${rel}_k$k=$? >> $S
  done
  SMA_MLP_RELAXPOLL=$rel SMA_MLP_PROF=3 timeout 300 python bench.py --config MLP --k 4 --steps 1000 --warmup 20 --rounds-per-call 1000 --no-cpu-baseline --no-e2e > gpurun_out/rp_prof_rel$rel.log 2>&1
done
timeout 1500 python -m pytest -q -x -rfs tests/test_gpu_parity.py -k "mlp" > gpurun_out/rp_pytest.log 2>&1; echo pytest=$? >> $S
echo done >> $S
