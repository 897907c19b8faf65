cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -rfs > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? > gpurun_out/status5.txt
