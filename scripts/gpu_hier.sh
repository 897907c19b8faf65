cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$? > gpurun_out/status_hier.txt
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -rfs -k "hierarch" > gpurun_out/pytest_hier.log 2>&1; echo hier=$? >> gpurun_out/status_hier.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rfs > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status_hier.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status_hier.txt
echo done >> gpurun_out/status_hier.txt
