# round 2, call U: small rounds (C2 LeNet k=8, C3 ResNet-32 k=16 at n = 1): rounds/s, kernel-only durations
# (launch list) and one ncu --set full capture of each (warm L2: --cache-control none)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_u.txt; : > $S
for c in C2 C3; do
  timeout 300 python bench.py --config $c --steps 5000 --warmup 100 --no-cpu-baseline --no-e2e > gpurun_out/u_bench_$c.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/u_launches_$c.csv python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  timeout 600 ncu --set full --import-source on --clock-control none --cache-control none -k regex:replica_step -s 50 -c 1 -o gpurun_out/u_ncu_$c python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/u_ncu_$c.log 2>&1
done
echo done >> $S
