cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/sg3.txt
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 900 -k "paper_config or mlp or randomized or synth_100 or hierarchical" > gpurun_out/pytest_sg3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/sg3.txt
for c in C1 MLP C2 C3 C5; do
    timeout 300 python bench.py --config $c --steps 3000 --no-cpu-baseline --no-e2e > gpurun_out/sg.log 2>&1
    echo "$c $(tail -1 gpurun_out/sg.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"]*1000,2))' 2>&1 | tail -1)" >> gpurun_out/sg3.txt
done
