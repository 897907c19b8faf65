cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rfs > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/status10.txt
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/status10.txt
for c in C1 MLP C2 C3 C5; do timeout 600 python bench.py --config $c --steps 500 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:replica_step -s 5 -c 2 -o gpurun_out/prof_ldg_full python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done >> gpurun_out/status10.txt
