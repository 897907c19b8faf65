cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/p2pgrid.txt
for k in 2 16; do for m in B A; do for v in 1 2 4; do
  SMA_P2P_CTAS_PER_SM=$v timeout 300 python bench.py --force-collective --mode $m --k $k --steps 500 --no-cpu-baseline --no-e2e > gpurun_out/pg.log 2>&1
  echo "k=$k mode=$m ctas/SM=$v $(tail -1 gpurun_out/pg.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); nv=d["nvlink"]; print(round(d["value"],1), round(d["ms_per_step"]*1000,1), "replica", round(d["roofline"]["avg_launch_ms"]*1000,1), "zsync", round(nv["fused_zsync_ms"]*1000,1))')" >> gpurun_out/p2pgrid.txt
done; done; done
