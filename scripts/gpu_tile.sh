cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/tile.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "learner or softmax or mlp" > gpurun_out/pytest_tile.log 2>&1; echo "pytest rc=$?" >> gpurun_out/tile.txt
for c in C1 MLP; do
  timeout 300 python bench.py --config $c --steps 3000 --no-cpu-baseline --no-e2e > gpurun_out/tl.log 2>&1
  echo "$c $(tail -1 gpurun_out/tl.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))')" >> gpurun_out/tile.txt
done
for c in C1 MLP; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 200 -c 40 --csv --log-file gpurun_out/tile_$c.csv python bench.py --config $c --steps 50 --warmup 100 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
