# round 2, call SV: softmax cluster kernel phase profile with the csync before dW split out (PROF build only)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
SMA_SOFTMAX_PROF=3 timeout 300 python bench.py --config C1 --steps 3000 --warmup 50 --rounds-per-call 1000 --no-cpu-baseline --no-e2e > gpurun_out/sv_prof.log 2>&1
echo done > gpurun_out/status_sv.txt
