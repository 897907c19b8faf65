# round 2, call T: per-GPU load of N = 8 emulated on one GPU (SMA_P2P_EMULATE_N=8): the C4 replica kernel with
# r = 2 and, concurrently in Mode B, a 1-rank z-sync moving one GPU's share of the 8-rank z-sync HBM traffic,
# paced by capping its grid; Mode A (serial) for the standalone z-sync time (calibration vs the ~116 us NVLink time)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_t.txt; : > $S
for c in 0 8 16 24 32 48; do for m in A B; do
  timeout 300 python bench.py --k 2 --force-collective --zsync p2p --mode $m --emulate-n 8 --emulate-ctas $c --steps 300 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/t_emu_c${c}_$m.log 2>&1
done; done
for m in A B; do
  timeout 300 python bench.py --k 2 --force-collective --zsync p2p --mode $m --steps 300 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/t_noemu_$m.log 2>&1
done
echo done >> $S
