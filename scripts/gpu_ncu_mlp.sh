cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:mlp_ --launch-skip 40 -c 4 -o gpurun_out/mlp_full -f python bench.py --config MLP --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_mlp.log 2>&1
echo ncu=$? >> gpurun_out/ncu_mlp.log
