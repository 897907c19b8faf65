cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 120 python scripts/probe_mc.py > gpurun_out/probe_mc.log 2>&1
nvidia-smi topo -m >> gpurun_out/probe_mc.log 2>&1
nvidia-smi nvlink -s -i 0 >> gpurun_out/probe_mc.log 2>&1
