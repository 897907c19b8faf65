cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/uj.txt
for c in C1 MLP C2 C3; do for v in "SMA_SPLIT_UJ=2" "SMA_SPLIT_UJ=4"; do
    env $v timeout 300 python bench.py --config $c --steps 3000 --no-cpu-baseline --no-e2e > gpurun_out/sg.log 2>&1
    echo "$c [$v] $(tail -1 gpurun_out/sg.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"]*1000,2))' 2>&1 | tail -1)" >> gpurun_out/uj.txt
done; done
for k in 16 32; do for v in "SMA_SPLIT_UJ=2" "SMA_SPLIT_UJ=4"; do
    env $v timeout 300 python bench.py --config C2 --k $k --steps 3000 --no-cpu-baseline --no-e2e > gpurun_out/sg.log 2>&1
    echo "C2 k=$k [$v] $(tail -1 gpurun_out/sg.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"]*1000,2))' 2>&1 | tail -1)" >> gpurun_out/uj.txt
done; done
