cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
rm -f gpurun_out/minb.txt
for mb in 1 4; do
  SMA_NVCC_EXTRA="-DSMA_SPLIT_MINB=$mb" python -c "from paper_1901_02244_b200 import _build; _build.build(force=True)" > gpurun_out/build.log 2>&1
  for c in C1 MLP C2 C3; do
    timeout 300 python bench.py --config $c --steps 3000 --no-cpu-baseline --no-e2e > gpurun_out/mb.log 2>&1
    echo "$c minb=$mb $(tail -1 gpurun_out/mb.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"]*1000,2))')" >> gpurun_out/minb.txt
  done
done
