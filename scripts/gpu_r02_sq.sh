# round 2, call SQ: the small-round floor -- host enqueue time per sma_step and the same rounds replayed
# from a CUDA graph of 100 captured steps (scripts/small_probe.py)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 400 python scripts/small_probe.py > gpurun_out/sq_probe.jsonl 2> gpurun_out/sq_probe.err; echo probe=$? > gpurun_out/status_sq.txt
