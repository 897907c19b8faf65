# round 2, call C (after the container restore): validate the committed state -- smoke, every GPU
# test, default bench, MLP fused-kernel bench, reference arm
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_c.txt; : > $S
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_c.log 2>&1; echo smoke=$? >> $S
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -rfs --durations=25 > gpurun_out/pytest_c.log 2>&1; echo pytest=$? >> $S
timeout 600 python bench.py > gpurun_out/bench_c4_c.log 2>&1; echo bench=$? >> $S
for k in 4 16; do
  timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/mlp_c_k$k.log 2>&1
done
echo done >> $S
