# SIMT layer-1 kernel: hidden units per CTA (SMA_MLP_HID_UNITS) at k = 4 / 8 (SIMT)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
out=gpurun_out/hid_units.txt; echo "# MLP rounds/s, SMA_MLP_TC=0, bench.py --config MLP --k K --steps 2000, SMA_MLP_HID_UNITS = U" > $out
for k in 4 8; do for u in 1 2 4 8 16; do
  v=$(SMA_MLP_TC=0 SMA_MLP_HID_UNITS=$u timeout 300 python bench.py --config MLP --k $k --steps 2000 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],1))")
  echo "MLP k=$k units=$u $v" >> $out; done; done
for u in 2 8; do SMA_MLP_HID_UNITS=$u timeout 600 python -m pytest tests -m gpu -q -k "mlp_gradient_single or mlp_learner_sma or tensor_cores" --timeout 600 > gpurun_out/pytest_hu$u.log 2>&1; echo "pytest units=$u rc=$?" >> $out; done
