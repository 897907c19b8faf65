# round 2 re-entry: the restored committed state on a fresh B200 -- smoke, every GPU test,
# the default bench line, the MLP lines, the C4 ncu launch list
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_re.txt; : > $S
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/re_smoke.log 2>&1; echo smoke=$? >> $S
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rfs > gpurun_out/re_pytest_gpu.log 2>&1; echo pytest=$? >> $S
timeout 600 python bench.py > gpurun_out/re_bench.log 2>&1; echo bench=$? >> $S
timeout 300 python bench.py --config MLP --k 4 --steps 3000 --warmup 50 --rounds-per-call 3000 --no-cpu-baseline --no-e2e > gpurun_out/re_mlp4.log 2>&1; echo mlp=$? >> $S
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/re_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/re_ncu.log 2>&1; echo ncu=$? >> $S
echo done >> $S
