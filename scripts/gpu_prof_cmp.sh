cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -s 6 -c 2 -o gpurun_out/prof_triad python scripts/triad_prof.py > gpurun_out/ncu_triad.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:replica_step_tma -s 3 -c 1 -o gpurun_out/prof_tma2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_tma2.log 2>&1
