cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/perm.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_p2p_multiprocess.py -m gpu -q -x --timeout 600 -k "learner or softmax or mlp or overlapped" > gpurun_out/pytest_perm.log 2>&1; echo "pytest rc=$?" >> gpurun_out/perm.txt
for st in 1000 3000; do for c in C1 MLP; do
  timeout 300 python bench.py --config $c --steps $st --no-cpu-baseline --no-e2e > gpurun_out/pm.log 2>&1
  echo "$c steps=$st $(tail -1 gpurun_out/pm.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))')" >> gpurun_out/perm.txt
done; done
timeout 600 python scripts/autotune_demo.py MLP > gpurun_out/autotune_MLP.jsonl 2>&1; echo "autotune rc=$?" >> gpurun_out/perm.txt

