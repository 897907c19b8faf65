cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
rm -f gpurun_out/ldg_policy.log
for rep in 1 2; do for pol in 0 1 2; do
  SMA_LDG_POLICY=$pol SWEEP_LDG_ONLY=1 timeout 300 python scripts/sweep.py 2>/dev/null | grep '^{' | sed "s/^/{\"policy\": $pol, \"rep\": $rep, \"r\": /; s/}$/}}/" >> gpurun_out/ldg_policy.log
done; done
