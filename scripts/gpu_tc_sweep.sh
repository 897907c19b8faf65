cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/tc_sweep.txt
for k in 2 4 6 8 12 16 32; do
  for tc in 0 1; do
    SMA_MLP_TC=$tc timeout 300 python bench.py --config MLP --k $k --steps 2000 --no-cpu-baseline --no-e2e > gpurun_out/sw_${k}_${tc}.log 2>&1
    echo "k=$k tc=$tc $(tail -1 gpurun_out/sw_${k}_${tc}.log | python -c 'import json,sys; print(json.loads(sys.stdin.read())["value"])')" >> gpurun_out/tc_sweep.txt
  done
done
