cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
rm -f gpurun_out/ldg_variants.log
for grid in persistent full; do for u in 2 4 8; do
  SMA_LDG_GRID=$grid SMA_LDG_UNROLL=$u SWEEP_LDG_ONLY=1 timeout 300 python scripts/sweep.py 2>/dev/null | grep '^{' | sed "s/^/{\"grid\": \"$grid\", \"unroll\": $u, \"r\": /; s/}$/}}/" >> gpurun_out/ldg_variants.log
done; done
SWEEP_TMA_ONLY=1 timeout 300 python scripts/sweep.py 2>/dev/null | grep '^{' | sed "s/^/{\"grid\": \"tma\", \"unroll\": 0, \"r\": /; s/}$/}}/" >> gpurun_out/ldg_variants.log
