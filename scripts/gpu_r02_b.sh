# round 2, call B: fused MLP kernel (tests, bench, ncu), pipelined ABI e2e, C4 default bench, P2P z-sync ncu at C3
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_b.txt; : > $S
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> $S
timeout 1500 python -m pytest -s -q --timeout 900 -rfs -k "mlp or pipelined or learner or errors" tests/test_gpu_parity.py > gpurun_out/pytest_b.log 2>&1; echo pytest=$? >> $S
for k in 4 8 12 16 32; do
  timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/mlp_fused_k$k.log 2>&1
  SMA_MLP_FUSED=0 timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/mlp_5k_k$k.log 2>&1
done
echo mlpbench=done >> $S
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.log 2>&1; echo bench=$? >> $S
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo ref=$? >> $S
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mlp_round_kernel -s 20 -c 1 -o gpurun_out/ncu_mlp_fused_k4 python bench.py --config MLP --k 4 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ncu_mlp.log 2>&1; echo ncu_mlp=$? >> $S
timeout 600 ncu --set full --import-source on --clock-control none -k regex:zsync_p2p -s 20 -c 1 -o gpurun_out/ncu_p2p_c3 python bench.py --config C3 --k 2 --force-collective --zsync p2p --mode A --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ncu_p2p.log 2>&1; echo ncu_p2p=$? >> $S
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_mlp_k4.csv python bench.py --config MLP --k 4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done >> $S
