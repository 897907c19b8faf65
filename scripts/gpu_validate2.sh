# gpu_validate.sh plus the MLP learner's default policy at k = 12 / 24 / 32
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash scripts/gpu_validate.sh
for k in 12 24 32; do timeout 300 python bench.py --config MLP --k $k --steps 2000 --no-cpu-baseline --no-e2e > gpurun_out/bench_MLP_k$k.log 2>&1; done
echo done2 >> gpurun_out/status_final.txt
