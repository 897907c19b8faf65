# MLP logits kernel with W2 staged before the PDL wait
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
out=gpurun_out/logits_prefetch.txt; echo "# MLP rounds/s, bench.py --config MLP --k K --steps 3000, default policy, logits kernel stages W2 before griddepcontrol.wait" > $out
timeout 900 python -m pytest tests -m gpu -q -k "mlp or learner" --timeout 600 > gpurun_out/pytest_lp.log 2>&1; echo "pytest rc=$?" >> $out; tail -1 gpurun_out/pytest_lp.log >> $out
for k in 4 8 16; do
  v=$(timeout 300 python bench.py --config MLP --k $k --steps 3000 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],1))")
  echo "MLP k=$k default $v" >> $out; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> $out
