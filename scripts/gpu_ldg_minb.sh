cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
rm -f gpurun_out/ldg_minb.log
for mb in 4 6 8; do
  SMA_LDG_MINB=$mb SWEEP_LDG_ONLY=1 timeout 300 python scripts/sweep.py 2>/dev/null | grep '^{' | sed "s/^/{\"minb\": $mb, \"r\": /; s/}$/}}/" >> gpurun_out/ldg_minb.log
done
