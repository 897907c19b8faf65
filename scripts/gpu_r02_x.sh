# round 2, call X: validation of the committed state -- build, smoke, every GPU test, the default bench (C4,
# N = 1, with cpu_baseline and e2e), the reference arm, the launch list and one ncu --set full capture of the
# headline kernel, and the other configs' lines
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_x.txt; : > $S
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/x_build.log 2>&1; echo build=$? >> $S
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/x_smoke.log 2>&1; echo smoke=$? >> $S
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rfs --durations=15 > gpurun_out/x_pytest_gpu.log 2>&1; echo pytest=$? >> $S
timeout 900 python bench.py > gpurun_out/x_bench_c4.log 2>&1; echo bench=$? >> $S
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/x_bench_ref.log 2>&1; echo ref=$? >> $S
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/x_launches_c4.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo launches=$? >> $S
timeout 900 ncu --set full --import-source on --clock-control none -k regex:replica_step -s 5 -c 1 -o gpurun_out/x_ncu_c4 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/x_ncu_c4.log 2>&1; echo ncu=$? >> $S
for c in C1 C2 C3 C5; do
  timeout 600 python bench.py --config $c --steps 2000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/x_bench_$c.log 2>&1
done
for k in 4 8 16 32; do
  timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --rounds-per-call 3000 --no-cpu-baseline --no-e2e > gpurun_out/x_mlp_multi_k$k.log 2>&1
  timeout 300 python bench.py --config MLP --k $k --steps 3000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/x_mlp_k$k.log 2>&1
done
echo done >> $S
