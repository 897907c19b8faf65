# round 2, calls SG, SI, SJ (SJ: producer warp decoupled by full/empty mbarriers): the softmax cluster kernel with st.async partial exchange (SI: reduce-scatter to row owners + e broadcast) and a producer warp --
# parity tests, C1 rates over M, phase profile
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_sj.txt; : > $S
timeout 900 python -m pytest -q -x -rfs tests/test_gpu_parity.py -k "softmax or learner_gradient_single or learner_step_fused or overlapped" > gpurun_out/sj_pytest.log 2>&1; echo pytest=$? >> $S
for M in 0 16 8 4; do
  for rpc in 1 1000; do
    SMA_SOFTMAX_M=$M timeout 300 python bench.py --config C1 --steps 3000 --warmup 50 --rounds-per-call $rpc --no-cpu-baseline --no-e2e > gpurun_out/sj_c1_m${M}_rpc$rpc.log 2>&1; echo c1_m${M}_$rpc=$? >> $S
  done
done
SMA_SOFTMAX_PROF=3 timeout 300 python bench.py --config C1 --steps 3000 --warmup 50 --rounds-per-call 1000 --no-cpu-baseline --no-e2e > gpurun_out/sj_prof.log 2>&1
echo done >> $S
