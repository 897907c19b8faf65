cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/c1.txt
for c in C1 MLP C2 C3; do
for v in "" "SMA_BENCH_GRAPH=1" "SMA_LEARNER_FUSE=0" "SMA_LEARNER_FUSE=0 SMA_BENCH_GRAPH=1"; do
  env $v timeout 300 python bench.py --config $c --steps 3000 --no-cpu-baseline --no-e2e > gpurun_out/c1.log 2>&1
  echo "$c [$v] $(tail -1 gpurun_out/c1.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"]*1000)' 2>&1 | tail -1)" >> gpurun_out/c1.txt
done; done
