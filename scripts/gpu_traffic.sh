cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for k in 16 8 4 2; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:replica_step -s 10 -c 2 --csv --log-file gpurun_out/traffic_B_k$k.csv python bench.py --force-collective --k $k --steps 5 --warmup 12 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  timeout 600 ncu --metrics $M --clock-control none -k regex:replica_step -s 10 -c 2 --csv --log-file gpurun_out/traffic_A_k$k.csv python bench.py --force-collective --mode A --k $k --steps 5 --warmup 12 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
timeout 600 ncu --metrics $M --clock-control none -k regex:replica_step -s 10 -c 2 --csv --log-file gpurun_out/traffic_fused_k16.csv python bench.py --steps 5 --warmup 12 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done > gpurun_out/status_traffic.txt
