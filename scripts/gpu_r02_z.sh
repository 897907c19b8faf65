# round 2, call Z: phase-1 K split independent of the warp-group sizes (multi-round == per-round bitwise again);
# MLP tests, MLP benches, compute-sanitizer on the fused MLP kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_z.txt; : > $S
timeout 1500 python -m pytest -q -rfs -k "mlp or learner" tests/test_gpu_parity.py > gpurun_out/z_pytest.log 2>&1; echo pytest=$? >> $S
for k in 4 8 16; do
  timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --rounds-per-call 3000 --no-cpu-baseline --no-e2e > gpurun_out/z_mlp_multi_k$k.log 2>&1
  timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/z_mlp_k$k.log 2>&1
done
CS=/usr/local/cuda/bin/compute-sanitizer
K="(mlp_learner_steps_multi_round_bitwise and (4 or 16)) or mlp_gradient_single_round or mlp_learner_sma_parity"
for tool in memcheck racecheck synccheck; do
  timeout 2400 $CS --tool $tool python -m pytest tests/test_gpu_parity.py -q -k "$K" > gpurun_out/z_san_$tool.log 2>&1; echo $tool=$? >> $S
done
echo done >> $S
