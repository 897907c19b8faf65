# round 2, call ST: the final softmax cluster kernel -- ncu --set full of one multi-round launch, and C1 rates over
# the slice count m (SMA_SOFTMAX_M = 16 default, 14, 12, 8)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_st.txt; : > $S
for M in 16 14 12 8; do
  SMA_SOFTMAX_M=$M timeout 300 python bench.py --config C1 --steps 3000 --warmup 50 --rounds-per-call 1000 --no-cpu-baseline --no-e2e > gpurun_out/st_m$M.log 2>&1; echo m$M=$? >> $S
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:softmax_cluster -s 2 -c 1 -o gpurun_out/st_softmax_cluster python bench.py --config C1 --steps 3000 --warmup 50 --rounds-per-call 1000 --no-cpu-baseline --no-e2e > gpurun_out/st_ncu.log 2>&1; echo ncu=$? >> $S
echo done >> $S
