# MLP learner: SIMT vs tensor-core GEMMs per layer over k (after the dW1 SIMT kernel's 4-wide register tile)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
out=gpurun_out/tc_sweep2.txt; echo "# MLP rounds/s, bench.py --config MLP --k K --steps 2000, SMA_MLP_TC = 0 (SIMT) / 1 (both TC) / hidden (layer 1 TC) / w1 (dW1 TC) / unset (default)" > $out
for k in 4 8 12 16 24 32; do for tc in 0 1 hidden w1 unset; do
  if [ $tc = unset ]; then v=$(timeout 300 python bench.py --config MLP --k $k --steps 2000 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],1))");
  else v=$(SMA_MLP_TC=$tc timeout 300 python bench.py --config MLP --k $k --steps 2000 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],1))"); fi
  echo "MLP k=$k tc=$tc $v" >> $out; done; done
timeout 900 python -m pytest tests -m gpu -q -k "mlp or learner" --timeout 600 > gpurun_out/pytest_tc2.log 2>&1; echo pytest=$? >> $out
