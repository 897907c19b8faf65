# round 2, call SO: softmax cluster kernel stress test (random call sizes, 600 rounds) and the softmax tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -rfs --durations=5 tests/test_gpu_parity.py -k "softmax" > gpurun_out/so_pytest.log 2>&1; echo pytest=$? > gpurun_out/status_so.txt
