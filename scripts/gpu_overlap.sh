cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? > gpurun_out/status_ov.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -rfs -k "overlapped or learner" > gpurun_out/pytest_ov.log 2>&1; echo ov=$? >> gpurun_out/status_ov.txt
for c in C1 MLP; do timeout 600 python bench.py --config $c --force-collective --steps 1000 --no-cpu-baseline --no-e2e > gpurun_out/bench_coll_$c.log 2>&1; done
echo done >> gpurun_out/status_ov.txt
