# round 2, call A: new parity tests at size / MLP bench configs / C ABI, P2P barrier + coherent loads
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_a.txt; : > $S
timeout 1500 python -m pytest -s -q --timeout 900 -rfs tests/test_gpu_parity_size.py "tests/test_gpu_parity.py::test_mlp_bench_configs_100_rounds" "tests/test_gpu_parity.py::test_mlp_learner_sma_parity" "tests/test_gpu_parity.py::test_learner_step_overlapped_zsync" tests/test_c_abi_program.py tests/test_p2p_multiprocess.py > gpurun_out/pytest_a.log 2>&1; echo pytest=$? >> $S
for bar in 0 1; do for m in A B; do
  SMA_P2P_BARRIER=$bar timeout 300 python bench.py --config C3 --k 2 --force-collective --zsync p2p --mode $m --steps 3000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/c3_bar${bar}_$m.log 2>&1
  SMA_P2P_BARRIER=$bar timeout 300 python bench.py --k 2 --force-collective --zsync p2p --mode $m --steps 300 --no-cpu-baseline --no-e2e > gpurun_out/c4_bar${bar}_$m.log 2>&1
done; done
echo bench=done >> $S
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --target-processes all --kernel-name regex:replica_step --csv --log-file gpurun_out/launches_size_tests.csv python -m pytest -q -x tests/test_gpu_parity_size.py > gpurun_out/ncu_size.log 2>&1; echo ncu=$? >> $S
