# round 2, calls SC/SD: the softmax learner's cluster kernel (sma_learner_softmax_fused.cu) -- parity tests
# (multi-round == per-round bitwise; vs the oracle) and C1 rates over the slice count M
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_sd.txt; : > $S
timeout 900 python -m pytest -q -x -rfs tests/test_gpu_parity.py -k "softmax or learner_gradient_single or learner_step_fused or overlapped" > gpurun_out/sd_pytest.log 2>&1; echo pytest=$? >> $S
for M in 0 16 14 8 7 4; do
  for rpc in 1 1000; do
    SMA_SOFTMAX_M=$M timeout 300 python bench.py --config C1 --steps 3000 --warmup 50 --rounds-per-call $rpc --no-cpu-baseline --no-e2e > gpurun_out/sd_c1_m${M}_rpc$rpc.log 2>&1; echo c1_m${M}_$rpc=$? >> $S
  done
done
echo done >> $S
