cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 500 -k "learner or softmax or mlp" > gpurun_out/pytest_c1b.log 2>&1; echo "pytest rc=$?" > gpurun_out/c1b.txt
timeout 300 python bench.py --config C1 --steps 3000 --no-cpu-baseline --no-e2e > gpurun_out/c1b.log 2>&1; tail -1 gpurun_out/c1b.log >> gpurun_out/c1b.txt
