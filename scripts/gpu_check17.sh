cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -rfs > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/status17.txt
timeout 300 python bench.py --force-collective --steps 300 --no-cpu-baseline --no-e2e > gpurun_out/bench_auto_coll.log 2>&1; echo autocoll=$? >> gpurun_out/status17.txt
timeout 300 python bench.py --force-collective --zsync nccl --steps 300 --no-cpu-baseline --no-e2e > gpurun_out/bench_nccl_coll.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/status17.txt
echo done >> gpurun_out/status17.txt
