# round 2, call SF: ncu --set full with source-level stall sampling of one multi-round launch of the softmax
# cluster kernel (C1, 1000 rounds per call)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:softmax_cluster -s 2 -c 1 -o gpurun_out/sf_softmax_cluster python bench.py --config C1 --steps 3000 --warmup 50 --rounds-per-call 1000 --no-cpu-baseline --no-e2e > gpurun_out/sf_ncu.log 2>&1
echo ncu=$? > gpurun_out/status_sf.txt
