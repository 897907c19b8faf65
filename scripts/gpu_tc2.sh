cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? > gpurun_out/status_tc2.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 500 -rfs -k "mlp" > gpurun_out/pytest_tc2.log 2>&1; echo tc=$? >> gpurun_out/status_tc2.txt
SMA_MLP_TC=1 timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python tests/mlp_grad_worker.py /tmp/g.npy 4 16 3 5 > gpurun_out/sanitizer_tc_memcheck.txt 2>&1; echo memcheck=$? >> gpurun_out/status_tc2.txt
SMA_MLP_TC=1 timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck python tests/mlp_grad_worker.py /tmp/g.npy 4 16 3 5 > gpurun_out/sanitizer_tc_racecheck.txt 2>&1; echo racecheck=$? >> gpurun_out/status_tc2.txt
SMA_MLP_TC=1 timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool synccheck python tests/mlp_grad_worker.py /tmp/g.npy 4 16 3 5 > gpurun_out/sanitizer_tc_synccheck.txt 2>&1; echo synccheck=$? >> gpurun_out/status_tc2.txt
echo done >> gpurun_out/status_tc2.txt
