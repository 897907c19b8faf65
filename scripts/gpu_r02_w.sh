# round 2, call W: measured L2-resident bandwidth (torch copy / add); split-kernel knobs at C2 / C3
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_w.txt; : > $S
timeout 300 python scripts/l2_peak.py > gpurun_out/w_l2_peak.json 2> gpurun_out/w_l2_peak.err; echo l2=$? >> $S
for c in C2 C3; do
  for g in 2 4 8; do for uj in 2 4; do
    SMA_SPLIT_G=$g SMA_SPLIT_UJ=$uj timeout 300 python bench.py --config $c --steps 5000 --warmup 100 --no-cpu-baseline --no-e2e > gpurun_out/w_${c}_g${g}_uj$uj.log 2>&1
  done; done
  SMA_SPLIT_BELOW=0 timeout 300 python bench.py --config $c --steps 5000 --warmup 100 --no-cpu-baseline --no-e2e > gpurun_out/w_${c}_ldg.log 2>&1
done
echo done >> $S
