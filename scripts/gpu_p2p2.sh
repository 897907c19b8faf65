cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -rfs -k "p2p" > gpurun_out/pytest_p2p1.log 2>&1; echo p2p1=$? > gpurun_out/status19.txt
timeout 1200 python -m pytest tests/test_p2p_multiprocess.py -q --timeout 300 -rfs -x > gpurun_out/pytest_p2pmp.log 2>&1; echo p2pmp=$? >> gpurun_out/status19.txt
timeout 300 python bench.py --force-collective --zsync p2p --steps 300 --no-cpu-baseline --no-e2e > gpurun_out/bench_p2pB.log 2>&1
echo done >> gpurun_out/status19.txt
