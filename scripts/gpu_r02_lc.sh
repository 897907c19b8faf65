# round 2, call LC: fused MLP kernel with learner clusters (the nblk unit blocks of a learner exchange partial
# logits through DSMEM with st.async; SMA_MLP_LC=1 vs 0) -- MLP parity tests, rates k = 4/8/16/32, profile k = 8
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_lc.txt; : > $S
timeout 1500 python -m pytest -q -x -rfs tests/test_gpu_parity.py -k "mlp" > gpurun_out/lc_pytest.log 2>&1; echo pytest=$? >> $S
for lc in 1 0; do
  for k in 4 8 16 32; do
    SMA_MLP_LC=$lc timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --rounds-per-call 3000 --no-cpu-baseline --no-e2e > gpurun_out/lc_lc${lc}_k$k.log 2>&1; echo lc${lc}_k$k=$? >> $S
    SMA_MLP_LC=$lc timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/lc_one_lc${lc}_k$k.log 2>&1
  done
  SMA_MLP_LC=$lc SMA_MLP_PROF=3 timeout 300 python bench.py --config MLP --k 8 --steps 1000 --warmup 20 --rounds-per-call 1000 --no-cpu-baseline --no-e2e > gpurun_out/lc_prof_lc$lc.log 2>&1
done
echo done >> $S
