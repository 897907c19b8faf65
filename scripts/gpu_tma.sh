cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 -rf -k "tma or fused" > gpurun_out/pytest_tma.log 2>&1; echo pytest=$? >> gpurun_out/status2.txt
timeout 600 python scripts/sweep.py > gpurun_out/sweep.log 2>&1; echo sweep=$? >> gpurun_out/status2.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:replica_step_tma -s 3 -c 1 -o gpurun_out/prof_tma python bench.py --tma --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_tma.log 2>&1
echo done >> gpurun_out/status2.txt
