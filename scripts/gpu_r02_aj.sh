# round 2, call AJ: phase-1 rows rg and rg + 8 per lane (conflict-free x loads), bound scale by multiplication -- MLP tests incl. cluster == flag
# protocol bitwise; default benches
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_aj.txt; : > $S
timeout 1500 python -m pytest -q -x -rfs -k "mlp or learner" tests/test_gpu_parity.py > gpurun_out/aj_pytest.log 2>&1; echo pytest=$? >> $S
for k in 4 8 16 32; do
  timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --rounds-per-call 3000 --no-cpu-baseline --no-e2e > gpurun_out/aj_multi_k$k.log 2>&1
  timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/aj_one_k$k.log 2>&1
done
echo done >> $S
SMA_MLP_PROF=3 timeout 300 python bench.py --config MLP --k 4 --steps 1000 --warmup 20 --rounds-per-call 1000 --no-cpu-baseline --no-e2e > gpurun_out/aj_prof_k4.log 2>&1
