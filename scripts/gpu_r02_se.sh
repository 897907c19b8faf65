# round 2, call SE: per-phase cycle profile of the softmax cluster kernel (SMA_SOFTMAX_PROF)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for M in 16 8; do
  SMA_SOFTMAX_M=$M SMA_SOFTMAX_PROF=3 timeout 300 python bench.py --config C1 --steps 3000 --warmup 50 --rounds-per-call 1000 --no-cpu-baseline --no-e2e > gpurun_out/se_prof_m$M.log 2>&1
done
echo done > gpurun_out/status_se.txt
