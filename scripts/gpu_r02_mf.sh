# round 2, call MF: ncu --set full --import-source of one multi-round launch of the FINAL fused MLP kernel (k = 4, b = 16 and classes = 10 compile-time) for the
# per-line stall / instruction breakdown of the dW1 + update phase
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mlp_round_kernel -s 2 -c 1 -o gpurun_out/mf_mlp python bench.py --config MLP --k 4 --steps 3000 --warmup 50 --rounds-per-call 1000 --no-cpu-baseline --no-e2e > gpurun_out/mf_ncu.log 2>&1
echo ncu=$? > gpurun_out/status_mf.txt
