# round 2, call LD: why the MLP learner clusters did not engage -- the occupancy query per k
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in 8 16 32; do
  SMA_MLP_LC_DEBUG=1 timeout 120 python bench.py --config MLP --k $k --steps 50 --warmup 5 --rounds-per-call 50 --no-cpu-baseline --no-e2e > gpurun_out/ld_k$k.log 2>&1
done
nvidia-smi -q | grep -i -A3 "gpc\|Multiprocessor" | head -20 > gpurun_out/ld_smi.txt
python -c "
import torch; p=torch.cuda.get_device_properties(0); print(p.multi_processor_count)" >> gpurun_out/ld_smi.txt
echo done > gpurun_out/status_ld.txt
