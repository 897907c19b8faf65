cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/pergpu.jsonl
for k in 16 8 4 2; do for m in A B; do
  timeout 300 python bench.py --force-collective --mode $m --k $k --steps 500 --no-cpu-baseline --no-e2e > gpurun_out/pg.log 2>&1
  tail -1 gpurun_out/pg.log >> gpurun_out/pergpu.jsonl
done; done
