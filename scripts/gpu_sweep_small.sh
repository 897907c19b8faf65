cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/sweep_small.log
for d in 7850 431080 464154 2000000; do
  for c in 0 2 4; do
    SWEEP_D=$d SWEEP_TMA_ONLY=1 SMA_TMA_CONFIG=$c timeout 300 python scripts/sweep.py 2>/dev/null | sed "s/^/{\"d\": $d, \"cfg\": $c, \"r\": /; s/}$/}}/" >> gpurun_out/sweep_small.log
  done
  SWEEP_D=$d SWEEP_LDG_ONLY=1 timeout 300 python scripts/sweep.py 2>/dev/null | sed "s/^/{\"d\": $d, \"cfg\": \"ldg\", \"r\": /; s/}$/}}/" >> gpurun_out/sweep_small.log
done
