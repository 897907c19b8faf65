# round 2, call SX (b = 16 and classes = 10 as compile-time constants): softmax cluster kernel with the z update and corrections moved into the partial-logit
# exchange's wait and the replica update merged into dW -- softmax tests, C1 rates, profile
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_sx.txt; : > $S
timeout 900 python -m pytest -q -x -rfs tests/test_gpu_parity.py -k "softmax or learner_gradient_single or nonfinite" > gpurun_out/sx_pytest.log 2>&1; echo pytest=$? >> $S
for rpc in 1 1000; do
  timeout 300 python bench.py --config C1 --steps 3000 --warmup 50 --rounds-per-call $rpc --no-cpu-baseline --no-e2e > gpurun_out/sx_c1_rpc$rpc.log 2>&1; echo c1_$rpc=$? >> $S
done
SMA_SOFTMAX_PROF=3 timeout 300 python bench.py --config C1 --steps 3000 --warmup 50 --rounds-per-call 1000 --no-cpu-baseline --no-e2e > gpurun_out/sx_prof.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sx_smoke.log 2>&1; echo smoke=$? >> $S
echo done >> $S
