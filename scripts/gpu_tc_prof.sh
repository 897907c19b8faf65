cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mlp_hidden -s 20 -c 1 -o gpurun_out/mlp_tc python bench.py --config MLP --steps 5 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/ncu_tc.log 2>&1; echo ncu=$? > gpurun_out/status_tcp.txt

