# round 2, call AH: MLP multi-round sweeps -- group-2 warps (SMA_MLP_ZWARPS 2/4) x units per CTA (SMA_MLP_U)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_ah.txt; : > $S
for k in 4 8; do for zw in 2 4; do for u in 0 16; do
  SMA_MLP_ZWARPS=$zw SMA_MLP_U=$u timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --rounds-per-call 3000 --no-cpu-baseline --no-e2e > gpurun_out/ah_k${k}_z${zw}_u$u.log 2>&1
done; done; done
echo done >> $S
