cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? > gpurun_out/status_tc.txt
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 250 -rfs -k "mlp" > gpurun_out/pytest_tc.log 2>&1; echo tc=$? >> gpurun_out/status_tc.txt
SMA_MLP_TC=0 timeout 300 python bench.py --config MLP --steps 2000 --no-cpu-baseline --no-e2e > gpurun_out/bench_mlp_simt.log 2>&1; echo simt=$? >> gpurun_out/status_tc.txt
timeout 300 python bench.py --config MLP --steps 2000 --no-cpu-baseline --no-e2e > gpurun_out/bench_mlp_tc.log 2>&1; echo bench=$? >> gpurun_out/status_tc.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 30 --csv --log-file gpurun_out/launches_mlp_tc.csv python bench.py --config MLP --steps 20 --warmup 20 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu=$? >> gpurun_out/status_tc.txt
echo done >> gpurun_out/status_tc.txt
