# round 2, call V: N = 8 per-GPU load emulation, pacing sweep around the NVLink-bound z-sync time (~116 us)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_v.txt; : > $S
for c in 64 96 128 160 224; do for m in A B; do
  timeout 300 python bench.py --k 2 --force-collective --zsync p2p --mode $m --emulate-n 8 --emulate-ctas $c --steps 300 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/v_emu_c${c}_$m.log 2>&1
done; done
for m in A B; do
  timeout 300 python bench.py --k 2 --force-collective --zsync p2p --push --mode $m --emulate-n 8 --steps 300 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/v_emu_push_$m.log 2>&1
done
echo done >> $S
