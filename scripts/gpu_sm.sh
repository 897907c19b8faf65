cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 500 -k "learner or softmax or mlp" > gpurun_out/pytest_sm.log 2>&1; echo "pytest rc=$?" > gpurun_out/sm.txt
for c in C1 MLP; do timeout 300 python bench.py --config $c --steps 3000 --no-cpu-baseline --no-e2e > gpurun_out/sm_$c.log 2>&1; echo "$c $(tail -1 gpurun_out/sm_$c.log | cut -c100-170)" >> gpurun_out/sm.txt; done
for c in C1 MLP; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 200 -c 40 --csv --log-file gpurun_out/small_$c.csv python bench.py --config $c --steps 50 --warmup 100 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
