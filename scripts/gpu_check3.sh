cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvidia-smi -q | grep -i -A3 "fabric\|nvlink" | head -30 > gpurun_out/fabric.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q --timeout 120 -rfs -k "nvls and dyadic and k0" -x > gpurun_out/pytest_nvls1.log 2>&1; echo nvls1=$? > gpurun_out/status4.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -rfs > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status4.txt
timeout 900 python scripts/sweep.py > gpurun_out/sweep_all2.log 2>&1; echo sweep=$? >> gpurun_out/status4.txt
timeout 300 python bench.py --force-collective --zsync nvls --mode A --steps 300 --no-cpu-baseline --no-e2e > gpurun_out/bench_nvlsA.log 2>&1
timeout 300 python bench.py --force-collective --zsync nvls --mode B --steps 300 --no-cpu-baseline --no-e2e > gpurun_out/bench_nvlsB.log 2>&1
echo done >> gpurun_out/status4.txt
