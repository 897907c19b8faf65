cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rfs > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/status9.txt
for c in C1 MLP; do timeout 600 python bench.py --config $c --steps 1000 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 40 --csv --log-file gpurun_out/launches_C1.csv python bench.py --config C1 --steps 50 --warmup 60 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done >> gpurun_out/status9.txt
