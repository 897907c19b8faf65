# round 2, call D: the k = 32 MLP per-round parity failure -- reproducible? fused kernel only?
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
S=gpurun_out/status_d.txt; : > $S
T="tests/test_gpu_parity.py::test_mlp_bench_configs_per_round_100_rounds"
timeout 300 python -m pytest -q -x "$T[32]" > gpurun_out/d_k32_a.log 2>&1; echo a=$? >> $S
timeout 300 python -m pytest -q -x "$T[32]" > gpurun_out/d_k32_b.log 2>&1; echo b=$? >> $S
SMA_MLP_FUSED=0 timeout 300 python -m pytest -q -x "$T[32]" > gpurun_out/d_k32_unfused.log 2>&1; echo unfused=$? >> $S
SMA_PDL=0 timeout 300 python -m pytest -q -x "$T[32]" > gpurun_out/d_k32_nopdl.log 2>&1; echo nopdl=$? >> $S
timeout 300 python scripts/debug_mlp_round.py 32 26 > gpurun_out/d_debug_26.log 2>&1; echo dbg=$? >> $S
echo done >> $S
