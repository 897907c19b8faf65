cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/pdl.txt
for c in C2 C3 C4 C1 MLP MLP16; do
  for v in "SMA_PDL=0" "SMA_PDL=1"; do
    st=3000; [ $c = C4 ] && st=500
    cc=$c; ex=""; [ $c = MLP16 ] && cc=MLP && ex="--k 16"
    env $v timeout 300 python bench.py --config $cc $ex --steps $st --no-cpu-baseline --no-e2e > gpurun_out/pdl.log 2>&1
    echo "$c [$v] $(tail -1 gpurun_out/pdl.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"]*1000,2))' 2>&1 | tail -1)" >> gpurun_out/pdl.txt
  done
done
SMA_MLP_TC=1 timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python tests/mlp_grad_worker.py /tmp/g.npy 4 16 3 5 > gpurun_out/san_pdl_mem.txt 2>&1; echo "memcheck rc=$? $(tail -1 gpurun_out/san_pdl_mem.txt)" >> gpurun_out/pdl.txt
SMA_MLP_TC=1 timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck python tests/mlp_grad_worker.py /tmp/g.npy 4 16 3 5 > gpurun_out/san_pdl_race.txt 2>&1; echo "racecheck rc=$? $(tail -1 gpurun_out/san_pdl_race.txt)" >> gpurun_out/pdl.txt
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_pdl.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pdl.txt
