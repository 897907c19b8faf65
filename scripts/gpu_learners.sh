cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/learners.txt
for c in C1 MLP C2 C3; do
  timeout 300 python bench.py --config $c --steps 3000 --no-cpu-baseline --no-e2e > gpurun_out/bl_$c.log 2>&1
  echo "$c $(tail -1 gpurun_out/bl_$c.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["avg_launch_ms"])')" >> gpurun_out/learners.txt
done
timeout 300 python bench.py --config MLP --k 16 --steps 2000 --no-cpu-baseline --no-e2e > gpurun_out/bl_MLP16.log 2>&1
echo "MLP16 $(tail -1 gpurun_out/bl_MLP16.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])')" >> gpurun_out/learners.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 500 -k "mlp or learner or softmax" > gpurun_out/pytest_l.log 2>&1; echo "pytest=$?" >> gpurun_out/learners.txt
