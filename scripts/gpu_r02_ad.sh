# round 2, call AD: cluster mode, z^{i+1} parts stored into every peer by DSMEM (no z TMA, no proxy fence); the r CTAs of a unit block form a cluster and compute
# z^{i+1} through DSMEM: no z slice, no ZD / P2 flags) -- MLP tests, benches (cluster on / off), profile
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_ad.txt; : > $S
timeout 1500 python -m pytest -q -x -rfs -k "mlp or learner" tests/test_gpu_parity.py > gpurun_out/ad_pytest.log 2>&1; echo pytest=$? >> $S
for cl in 1 0; do for k in 4 8 16; do
  SMA_MLP_CLUSTER=$cl timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --rounds-per-call 3000 --no-cpu-baseline --no-e2e > gpurun_out/ad_multi_cl${cl}_k$k.log 2>&1
  SMA_MLP_CLUSTER=$cl timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/ad_one_cl${cl}_k$k.log 2>&1
done; done
for k in 4 8; do
SMA_MLP_PROF=3 timeout 300 python bench.py --config MLP --k $k --steps 1000 --warmup 20 --rounds-per-call 1000 --no-cpu-baseline --no-e2e > gpurun_out/ad_prof_k$k.log 2>&1
done
echo done >> $S
