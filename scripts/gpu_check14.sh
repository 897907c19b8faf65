cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench.py --force-collective --steps 200 --no-cpu-baseline --no-e2e > gpurun_out/bench_collB.log 2>&1; echo collB=$? > gpurun_out/status14.txt
timeout 600 python bench.py --tau 0 --steps 500 --no-cpu-baseline --no-e2e > gpurun_out/bench_tau0.log 2>&1; echo tau0=$? >> gpurun_out/status14.txt
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$? >> gpurun_out/status14.txt
echo done >> gpurun_out/status14.txt
