# round 2, calls SM (1|2|4 scalar e loads), SN (4|8 float4 e loads): softmax cluster kernel, dW item granularity (SMA_SOFTMAX_GQ = classes per thread item)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_sn.txt; : > $S
for gq in 4 8; do
  SMA_SOFTMAX_GQ=$gq timeout 300 python bench.py --config C1 --steps 3000 --warmup 50 --rounds-per-call 1000 --no-cpu-baseline --no-e2e > gpurun_out/sn_gq$gq.log 2>&1; echo gq$gq=$? >> $S
  SMA_SOFTMAX_GQ=$gq SMA_SOFTMAX_PROF=3 timeout 300 python bench.py --config C1 --steps 3000 --warmup 50 --rounds-per-call 1000 --no-cpu-baseline --no-e2e > gpurun_out/sn_prof_gq$gq.log 2>&1
done
SMA_SOFTMAX_GQ=8 timeout 600 python -m pytest -q -x tests/test_gpu_parity.py -k "softmax_cluster" > gpurun_out/sn_pytest.log 2>&1; echo pytest=$? >> $S
echo done >> $S
