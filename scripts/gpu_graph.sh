cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/graph.txt
for c in C2 C3 C4; do for v in "" "SMA_BENCH_GRAPH=1" "" "SMA_BENCH_GRAPH=1"; do
  st=3000; [ $c = C4 ] && st=500
  env $v timeout 300 python bench.py --config $c --steps $st --no-cpu-baseline --no-e2e > gpurun_out/gr.log 2>&1
  echo "$c [$v] $(tail -1 gpurun_out/gr.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"]*1000,2))')" >> gpurun_out/graph.txt
done; done
