cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in C2 C3; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 100 -c 40 --csv --log-file gpurun_out/small_$c.csv python bench.py --config $c --steps 50 --warmup 100 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
