# round-end check (tests only): build, smoke, every GPU test
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? > gpurun_out/status_final2.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status_final2.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rfs > gpurun_out/pytest_gpu_final2.log 2>&1; echo pytest=$? >> gpurun_out/status_final2.txt
