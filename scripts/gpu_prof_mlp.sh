cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --cache-control none -k regex:"mlp_hidden_kernel|mlp_w1_kernel" -s 20 -c 2 -o gpurun_out/mlp_simt2 python bench.py --config MLP --steps 5 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/ncu_mlp2.log 2>&1; echo rc=$? > gpurun_out/status_pm.txt
