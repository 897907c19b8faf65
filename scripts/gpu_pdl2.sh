cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/pdl2.txt
for v in "SMA_LEARNER_FUSE=0" "SMA_LEARNER_FUSE=1"; do
  env $v timeout 300 python bench.py --config C1 --steps 3000 --no-cpu-baseline --no-e2e > gpurun_out/p2.log 2>&1
  echo "C1 [$v] $(tail -1 gpurun_out/p2.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))')" >> gpurun_out/pdl2.txt
done
for k in 4 6 8 12 16 32; do for tc in 0 1; do
  SMA_MLP_TC=$tc timeout 300 python bench.py --config MLP --k $k --steps 2000 --no-cpu-baseline --no-e2e > gpurun_out/p2.log 2>&1
  echo "MLP k=$k tc=$tc $(tail -1 gpurun_out/p2.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))')" >> gpurun_out/pdl2.txt
done; done
