# round 2, call M: (1) C3 k=2 per-GPU round with the 1-rank P2P z-sync, barrier variants (SMA_P2P_BARRIER=0: every
# CTA acquires at system scope + per-CTA __threadfence_system; 1: one CTA + gpu-scope arrivals), Modes A/B;
# (2) the launch list of the at-size parity tests (which replica_step_ldg instantiations they run)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_m.txt; : > $S
for bar in 0 1; do for m in A B; do
  SMA_P2P_BARRIER=$bar timeout 300 python bench.py --config C3 --k 2 --force-collective --zsync p2p --mode $m --steps 5000 --warmup 100 --no-cpu-baseline --no-e2e > gpurun_out/m_c3_bar${bar}_$m.log 2>&1
done; done
echo bench=done >> $S
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --target-processes all --kernel-name regex:replica_step --csv --log-file gpurun_out/m_launches_size_tests.csv python -m pytest -q -x tests/test_gpu_parity_size.py > gpurun_out/m_ncu_size.log 2>&1; echo ncu=$? >> $S
echo done >> $S
