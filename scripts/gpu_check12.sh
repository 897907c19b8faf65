cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rfs > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/status12.txt
rm -f gpurun_out/split.log
for sb in 0 151552; do for d in 7850 431080 464154; do
  SMA_SPLIT_BELOW=$sb SWEEP_D=$d SWEEP_LDG_ONLY=1 timeout 300 python scripts/sweep.py 2>/dev/null | grep '^{' | sed "s/^/{\"split_below\": $sb, \"d\": $d, \"r\": /; s/}$/}}/" >> gpurun_out/split.log
done; done
for c in C2 C3; do timeout 600 python bench.py --config $c --steps 1000 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1; done
echo done >> gpurun_out/status12.txt
