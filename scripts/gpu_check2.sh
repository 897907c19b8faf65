cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/status3.txt
timeout 600 python scripts/sweep.py > gpurun_out/sweep_all.log 2>&1
for c in 1 2 3 4 5 6; do SWEEP_TMA_ONLY=1 SMA_TMA_CONFIG=$c timeout 300 python scripts/sweep.py >> gpurun_out/sweep_tma.log 2>&1; done
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/status3.txt
timeout 300 python bench.py --force-collective --mode B --steps 300 --no-cpu-baseline --no-e2e > gpurun_out/bench_collB.log 2>&1
echo done >> gpurun_out/status3.txt
