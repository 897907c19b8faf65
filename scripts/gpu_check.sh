set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/status.txt
timeout 300 python bench.py --force-collective --mode A --steps 300 --no-cpu-baseline > gpurun_out/bench_collA.log 2>&1
timeout 300 python bench.py --force-collective --mode B --steps 300 --no-cpu-baseline > gpurun_out/bench_collB.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:replica_step -s 5 -c 2 -o gpurun_out/prof_c4 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
echo done >> gpurun_out/status.txt
