cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; python scripts/hbm_mix.py > gpurun_out/hbm_mix.json 2>&1
