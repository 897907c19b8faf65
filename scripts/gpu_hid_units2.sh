# SIMT layer-1 kernel with the one-wave hidden-units rule (default) vs forced units; SIMT vs TC at k = 12 / 16
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
out=gpurun_out/hid_units2.txt; echo "# MLP rounds/s, bench.py --config MLP --k K --steps 2000; default policy (one-wave units rule; layer 1 on tcgen05 from r >= 12) and SMA_MLP_TC=0" > $out
timeout 900 python -m pytest tests -m gpu -q -k "mlp or learner" --timeout 600 > gpurun_out/pytest_hu.log 2>&1; echo "pytest rc=$?" >> $out
for k in 2 4 8 12 16; do for tc in unset 0; do
  if [ $tc = unset ]; then v=$(timeout 300 python bench.py --config MLP --k $k --steps 2000 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],1))");
  else v=$(SMA_MLP_TC=0 timeout 300 python bench.py --config MLP --k $k --steps 2000 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],1))"); fi
  echo "MLP k=$k tc=$tc $v" >> $out; done; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> $out
