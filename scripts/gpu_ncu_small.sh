cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --cache-control none -k regex:replica_step_split -s 50 -c 1 -o gpurun_out/ncu_c2_split python bench.py --config C2 --steps 20 --warmup 60 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:zsync_p2p -s 5 -c 1 -o gpurun_out/ncu_p2p python bench.py --force-collective --mode A --steps 10 --warmup 8 --no-cpu-baseline --no-e2e > gpurun_out/ncu_p2p.log 2>&1
echo done > gpurun_out/status_ncus.txt
