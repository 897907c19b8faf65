cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? > gpurun_out/status_final.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status_final.txt
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rfs > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status_final.txt
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/status_final.txt
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$? >> gpurun_out/status_final.txt
for c in C1 MLP C2 C3 C5; do st=3000; [ $c = C5 ] && st=300; timeout 600 python bench.py --config $c --steps $st --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1; done
timeout 600 python bench.py --config MLP --k 16 --steps 3000 --no-cpu-baseline --no-e2e > gpurun_out/bench_MLP16.log 2>&1
timeout 600 python bench.py --force-collective --steps 300 --no-cpu-baseline --no-e2e > gpurun_out/bench_coll_p2p.log 2>&1
timeout 600 python bench.py --force-collective --zsync nccl --steps 300 --no-cpu-baseline --no-e2e > gpurun_out/bench_coll_nccl.log 2>&1
timeout 600 python scripts/autotune_demo.py MLP > gpurun_out/autotune_MLP.jsonl 2>&1; echo autotune=$? >> gpurun_out/status_final.txt
timeout 600 python scripts/autotune_demo.py C1 > gpurun_out/autotune_C1.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done >> gpurun_out/status_final.txt
