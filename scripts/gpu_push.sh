cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/push.txt
timeout 2400 python -m pytest tests/test_p2p_multiprocess.py tests/test_gpu_parity.py -m gpu -q -x --timeout 900 -k "push" > gpurun_out/pytest_push.log 2>&1; echo "pytest rc=$?" >> gpurun_out/push.txt
for k in 16 2; do for m in A B; do for p in "" "--push"; do
  timeout 300 python bench.py --force-collective --mode $m --k $k $p --steps 500 --no-cpu-baseline --no-e2e > gpurun_out/ps.log 2>&1
  echo "k=$k mode=$m [$p] $(tail -1 gpurun_out/ps.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); nv=d["nvlink"]; print(round(d["value"],1), "replica", round(d["roofline"]["avg_launch_ms"]*1000,1), "zsync", round(nv["fused_zsync_ms"]*1000,1))')" >> gpurun_out/push.txt
done; done; done
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --target-processes all python -m pytest tests/test_p2p_multiprocess.py -q -x -k "push_equals_pull_bitwise and 3-7 and A" > gpurun_out/san_push.log 2>&1; echo "memcheck rc=$? $(grep 'ERROR SUMMARY' gpurun_out/san_push.log | tail -1)" >> gpurun_out/push.txt
