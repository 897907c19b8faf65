cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/pdl3.txt
for c in C3; do for m in A B; do for z in p2p; do for v in "SMA_PDL=0" "SMA_PDL=1"; do
  st=2000; [ $c = C4 ] && st=300
  env $v timeout 300 python bench.py --config $c --force-collective --mode $m --zsync $z --steps $st --no-cpu-baseline --no-e2e > gpurun_out/p3.log 2>&1
  echo "$c mode=$m $z [$v] $(tail -1 gpurun_out/p3.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"]*1000,2))')" >> gpurun_out/pdl3.txt
done; done; done; done

