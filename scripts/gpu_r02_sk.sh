# round 2, call SK: the softmax cluster kernel final form -- parity tests, C1 rates (one round per call /
# the rounds of an epoch per call), compute-sanitizer memcheck + racecheck + synccheck on its tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_sk.txt; : > $S
timeout 900 python -m pytest -q -x -rfs tests/test_gpu_parity.py -k "softmax or learner_gradient_single or learner_step_fused or overlapped or randomized" > gpurun_out/sk_pytest.log 2>&1; echo pytest=$? >> $S
for rpc in 1 1000; do
  timeout 300 python bench.py --config C1 --steps 3000 --warmup 50 --rounds-per-call $rpc --no-cpu-baseline --no-e2e > gpurun_out/sk_c1_rpc$rpc.log 2>&1; echo c1_$rpc=$? >> $S
done
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest -q -x tests/test_gpu_parity.py -k "softmax_cluster_rounds and 784-10-16-4 or softmax_cluster_rounds and 40-16-7-5" > gpurun_out/sk_sanitizer_$tool.txt 2>&1; echo $tool=$? >> $S
done
echo done >> $S
