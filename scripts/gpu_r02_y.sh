# round 2, call Y: compute-sanitizer on the fused MLP kernel (multi-round launches with the per-CTA flag
# protocol, k = 4 and 16; the gradient-only instantiation through sma_learner_grads)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_y.txt; : > $S
CS=/usr/local/cuda/bin/compute-sanitizer
K="(mlp_learner_steps_multi_round_bitwise and (4 or 16)) or mlp_gradient_single_round"
for tool in memcheck racecheck synccheck; do
  timeout 2400 $CS --tool $tool python -m pytest tests/test_gpu_parity.py -q -x -k "$K" > gpurun_out/y_san_$tool.log 2>&1; echo $tool=$? >> $S
done
echo done >> $S
# the full-grid LDG kernel with more replicas in flight per thread at the small sizes (instead of the split kernel)
for c in C2 C3; do for u in 4 8; do
  SMA_SPLIT_BELOW=0 SMA_LDG_UNROLL=$u timeout 300 python bench.py --config $c --steps 5000 --warmup 100 --no-cpu-baseline --no-e2e > gpurun_out/y_${c}_ldg_u$u.log 2>&1
done; done
echo done2 >> $S
