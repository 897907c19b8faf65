# MLP default policy after the wave-fill rule (SIMT layer 1 when its grid fills >= 85 % of one wave)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
out=gpurun_out/hid_units3.txt; echo "# MLP rounds/s, bench.py --config MLP --k K --steps 2000, default policy (wave-fill rule)" > $out
timeout 900 python -m pytest tests -m gpu -q -k "mlp or learner" --timeout 600 > gpurun_out/pytest_hu3.log 2>&1; echo "pytest rc=$?" >> $out
for k in 4 8 12 16 24 32; do
  v=$(timeout 300 python bench.py --config MLP --k $k --steps 2000 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],1))")
  echo "MLP k=$k default $v" >> $out; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> $out
timeout 600 python bench.py > gpurun_out/bench_final.log 2>&1; echo "bench rc=$?" >> $out
