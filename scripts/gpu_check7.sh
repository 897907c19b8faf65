cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
# memory / race / sync checks of the hot-path kernels on small cases
timeout 900 compute-sanitizer --tool memcheck --leak-check full python -m pytest tests/test_gpu_parity.py -q -x -k "dyadic and (fused or collA or collB or matc) and not nvls" > gpurun_out/sanitizer_memcheck.log 2>&1; echo memcheck=$? > gpurun_out/status7.txt
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -q -x -k "synth_100_rounds_parity and 4097 and (fused_tma or matc_tma or fused-)" > gpurun_out/sanitizer_racecheck.log 2>&1; echo racecheck=$? >> gpurun_out/status7.txt
timeout 900 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_parity.py -q -x -k "synth_100_rounds_parity and 4097 and (fused_tma or matc)" > gpurun_out/sanitizer_synccheck.log 2>&1; echo synccheck=$? >> gpurun_out/status7.txt
# launch lists for the learner configs and the collective path
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 60 --csv --log-file gpurun_out/launches_C1.csv python bench.py --config C1 --steps 50 --warmup 60 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 60 --csv --log-file gpurun_out/launches_MLP.csv python bench.py --config MLP --steps 50 --warmup 60 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 40 --csv --log-file gpurun_out/launches_collB.csv python bench.py --force-collective --k 2 --steps 20 --warmup 10 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/status7.txt
for c in C1 MLP C2 C3; do timeout 600 python bench.py --config $c --steps 300 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1; done
echo done >> gpurun_out/status7.txt
