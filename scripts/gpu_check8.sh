cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -rfs -k "learner or mlp or softmax" > gpurun_out/pytest_learner.log 2>&1; echo pytest=$? > gpurun_out/status8.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 60 --csv --log-file gpurun_out/launches_C1.csv python bench.py --config C1 --steps 50 --warmup 60 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 60 --csv --log-file gpurun_out/launches_MLP.csv python bench.py --config MLP --steps 50 --warmup 60 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mlp_" -s 20 -c 3 -o gpurun_out/prof_learners python bench.py --config MLP --steps 10 --warmup 5 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"softmax_grad" -s 10 -c 1 -o gpurun_out/prof_softmax python bench.py --config C1 --steps 10 --warmup 5 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for c in C1 MLP; do timeout 600 python bench.py --config $c --steps 300 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1; done
echo done >> gpurun_out/status8.txt
