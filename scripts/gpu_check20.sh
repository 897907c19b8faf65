cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rfs -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/status20.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mlp_" -s 20 -c 3 -o gpurun_out/prof_mlp2 python bench.py --config MLP --steps 10 --warmup 5 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done >> gpurun_out/status20.txt
