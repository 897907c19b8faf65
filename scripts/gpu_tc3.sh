cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? > gpurun_out/status_tc3.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 500 -rfs -k "mlp" > gpurun_out/pytest_tc3.log 2>&1; echo tc=$? >> gpurun_out/status_tc3.txt
SMA_MLP_TC=1 timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python tests/mlp_grad_worker.py /tmp/g.npy 4 16 3 5 > gpurun_out/sanitizer_tc_memcheck.txt 2>&1; echo memcheck=$? >> gpurun_out/status_tc3.txt
SMA_MLP_TC=1 timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck python tests/mlp_grad_worker.py /tmp/g.npy 4 16 3 5 > gpurun_out/sanitizer_tc_racecheck.txt 2>&1; echo racecheck=$? >> gpurun_out/status_tc3.txt
SMA_MLP_TC=1 timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool synccheck python tests/mlp_grad_worker.py /tmp/g.npy 4 16 3 5 > gpurun_out/sanitizer_tc_synccheck.txt 2>&1; echo synccheck=$? >> gpurun_out/status_tc3.txt
rm -f gpurun_out/tc_sweep.txt
for k in 2 4 8 16 32; do
  for tc in 0 1; do
    SMA_MLP_TC=$tc timeout 300 python bench.py --config MLP --k $k --steps 2000 --no-cpu-baseline --no-e2e > gpurun_out/sw_${k}_${tc}.log 2>&1
    echo "k=$k tc=$tc $(tail -1 gpurun_out/sw_${k}_${tc}.log | python -c 'import json,sys; print(json.loads(sys.stdin.read())["value"])')" >> gpurun_out/tc_sweep.txt
  done
done
SMA_MLP_TC=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 30 --csv --log-file gpurun_out/launches_mlp_tc.csv python bench.py --config MLP --steps 20 --warmup 20 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done >> gpurun_out/status_tc3.txt
