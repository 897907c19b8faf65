# round 2, call AG: R18 certainty threshold 2^-15 (rigorous for the 12-slice sum) instead of 2^-12 -- MLP tests incl. cluster == flag
# protocol bitwise; default benches
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_ag.txt; : > $S
timeout 1500 python -m pytest -q -x -rfs -k "mlp or learner" tests/test_gpu_parity.py > gpurun_out/ag_pytest.log 2>&1; echo pytest=$? >> $S
for k in 4 8 16 32; do
  timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --rounds-per-call 3000 --no-cpu-baseline --no-e2e > gpurun_out/ag_multi_k$k.log 2>&1
  timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/ag_one_k$k.log 2>&1
done
echo done >> $S
