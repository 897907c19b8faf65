cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/pdl4.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "mlp" > gpurun_out/pytest_pdl4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pdl4.txt
for c in MLP16 MLP16b MLP; do
  cc=$c; ex=""; case $c in MLP16*) cc=MLP; ex="--k 16";; esac
  timeout 300 python bench.py --config $cc $ex --steps 3000 --no-cpu-baseline --no-e2e > gpurun_out/p4.log 2>&1
  echo "$c $(tail -1 gpurun_out/p4.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))')" >> gpurun_out/pdl4.txt
done
SMA_MLP_TC=1 timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck python tests/mlp_grad_worker.py /tmp/g.npy 4 16 3 5 > gpurun_out/san4.txt 2>&1; echo "racecheck rc=$? $(tail -1 gpurun_out/san4.txt)" >> gpurun_out/pdl4.txt
SMA_MLP_TC=0 timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python tests/mlp_grad_worker.py /tmp/g.npy 4 16 3 5 > gpurun_out/san4m.txt 2>&1; echo "memcheck rc=$? $(tail -1 gpurun_out/san4m.txt)" >> gpurun_out/pdl4.txt
