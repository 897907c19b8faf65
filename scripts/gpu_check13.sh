cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rfs > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/status13.txt
for c in C1 C2 C3; do timeout 600 python bench.py --config $c --steps 1000 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1; done
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/status13.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status13.txt
echo done >> gpurun_out/status13.txt
