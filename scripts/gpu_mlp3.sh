cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
echo skip > gpurun_out/m3.txt
for k in 10 12 16; do for tc in 0 1; do
SMA_MLP_TC=$tc timeout 300 python bench.py --config MLP --k $k --steps 3000 --no-cpu-baseline --no-e2e > gpurun_out/m3.log 2>&1; echo "MLP k=$k tc=$tc $(tail -1 gpurun_out/m3.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))')" >> gpurun_out/m3.txt
done; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:mlp_hidden -s 20 -c 5 --csv --log-file gpurun_out/m3.csv python bench.py --config MLP --steps 20 --warmup 20 --no-cpu-baseline --no-e2e > /dev/null 2>&1
