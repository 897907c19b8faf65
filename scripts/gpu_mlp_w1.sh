cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? > gpurun_out/status_w1.txt
timeout 900 python -m pytest tests -m gpu -q -k "mlp or learner" --timeout 600 > gpurun_out/pytest_w1.log 2>&1; echo pytest=$? >> gpurun_out/status_w1.txt
for k in 4 8 16; do for tc in 0 1; do SMA_MLP_TC=$tc timeout 300 python bench.py --config MLP --k $k --steps 3000 --no-cpu-baseline --no-e2e > gpurun_out/w1_k${k}_tc$tc.log 2>&1; done; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_w1.csv python bench.py --config MLP --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:mlp_w1 --launch-skip 10 -c 1 -o gpurun_out/w1_full -f python bench.py --config MLP --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done >> gpurun_out/status_w1.txt
