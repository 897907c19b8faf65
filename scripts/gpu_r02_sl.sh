# round 2, call SL: the final softmax cluster kernel -- ncu --set full (source stalls) of one multi-round launch,
# the non-finite tests on the fused learner kernels, the C1 bench lines
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_sl.txt; : > $S
timeout 900 python -m pytest -q -x -rfs tests/test_gpu_parity.py -k "nonfinite or softmax or learner_steps" > gpurun_out/sl_pytest.log 2>&1; echo pytest=$? >> $S
for rpc in 1 1000; do
  timeout 300 python bench.py --config C1 --steps 3000 --warmup 50 --rounds-per-call $rpc --no-cpu-baseline --no-e2e > gpurun_out/sl_c1_rpc$rpc.log 2>&1; echo c1_$rpc=$? >> $S
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:softmax_cluster -s 2 -c 1 -o gpurun_out/sl_softmax_cluster python bench.py --config C1 --steps 3000 --warmup 50 --rounds-per-call 1000 --no-cpu-baseline --no-e2e > gpurun_out/sl_ncu.log 2>&1; echo ncu=$? >> $S
echo done >> $S
