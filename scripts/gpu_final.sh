# round-end check: build, smoke, the whole GPU test suite, the default bench line, the MLP configs
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? > gpurun_out/status_final.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status_final.txt
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -rfs > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status_final.txt
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/status_final.txt
timeout 300 python bench.py --config MLP --steps 3000 --no-cpu-baseline --no-e2e > gpurun_out/bench_MLP.log 2>&1
timeout 300 python bench.py --config MLP --k 16 --steps 3000 --no-cpu-baseline --no-e2e > gpurun_out/bench_MLP16.log 2>&1
echo done >> gpurun_out/status_final.txt
