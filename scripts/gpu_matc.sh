cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "matc" > gpurun_out/pytest_matc.log 2>&1; echo pytest=$? > gpurun_out/status15.txt
timeout 300 python bench.py --matc --steps 300 --no-cpu-baseline --no-e2e > gpurun_out/bench_matc.log 2>&1
timeout 300 python bench.py --matc --k 2 --steps 300 --no-cpu-baseline --no-e2e > gpurun_out/bench_matc_k2.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 10 -c 20 --csv --log-file gpurun_out/launches_matc.csv python bench.py --matc --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done >> gpurun_out/status15.txt
