# round 2, call SP: small-round floor -- per-round time vs d (scripts/small_probe.py), the split
# kernel with a 6 / 8 CTA-per-SM register budget (SMA_SPLIT_MINB_RT), and a warm-L2 ncu launch
# list of C2 / C3 rounds (kernel duration vs round time)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_sp.txt; : > $S
timeout 300 python scripts/small_probe.py > gpurun_out/sp_probe.jsonl 2> gpurun_out/sp_probe.err; echo probe=$? >> $S
for m in 6 8; do
  SMA_SPLIT_MINB_RT=$m timeout 300 python scripts/small_probe.py > gpurun_out/sp_probe_minb$m.jsonl 2>&1; echo minb$m=$? >> $S
done
for c in C2 C3; do
  timeout 300 python bench.py --config $c --steps 5000 --warmup 100 --no-cpu-baseline --no-e2e > gpurun_out/sp_bench_$c.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum.per_second --clock-control none --cache-control none -c 60 -s 500 --csv --log-file gpurun_out/sp_ncu_$c.csv python bench.py --config $c --steps 600 --warmup 10 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu_$c=$? >> $S
done
echo done >> $S
