cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python scripts/autotune_demo.py C1 2000 30 > gpurun_out/autotune_C1.jsonl 2>&1
timeout 600 python scripts/autotune_demo.py MLP 500 24 > gpurun_out/autotune_MLP.jsonl 2>&1
for t in 1 4 0; do timeout 600 python bench.py --tau $t --steps 1000 --no-cpu-baseline --no-e2e > gpurun_out/bench_tau$t.log 2>&1; done
SWEEP_LDG_ONLY=1 timeout 300 python scripts/sweep.py > gpurun_out/sweep_prio.log 2>&1
echo done > gpurun_out/status11.txt
