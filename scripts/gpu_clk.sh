cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/clk.txt
for c in C1 C2 MLP; do for st in 1000 3000; do
  timeout 300 python bench.py --config $c --steps $st --no-cpu-baseline --no-e2e > gpurun_out/ck.log 2>&1
  echo "$c $st $(tail -1 gpurun_out/ck.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), d["clocks"])')" >> gpurun_out/clk.txt
done; done
timeout 300 python bench.py --steps 1000 --no-cpu-baseline --no-e2e > gpurun_out/ck.log 2>&1
echo "C4 1000 $(tail -1 gpurun_out/ck.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), d["clocks"])')" >> gpurun_out/clk.txt
