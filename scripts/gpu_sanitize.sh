cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -q -x -k "(dyadic or synth_100_rounds_parity) and not nvls and not 100003" > gpurun_out/sanitizer_memcheck.log 2>&1; echo memcheck=$? > gpurun_out/status18.txt
timeout 1200 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -q -x -k "(synth_100_rounds_parity and 4097 and (p2p or matc or fused)) or learner_step_fused or mlp_gradient_single or learner_gradient_single" > gpurun_out/sanitizer_racecheck.log 2>&1; echo racecheck=$? >> gpurun_out/status18.txt
timeout 1200 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_parity.py -q -x -k "(synth_100_rounds_parity and 4097 and (p2p or matc or tma)) or learner_step_fused or mlp_gradient_single" > gpurun_out/sanitizer_synccheck.log 2>&1; echo synccheck=$? >> gpurun_out/status18.txt
timeout 1200 compute-sanitizer --tool memcheck --target-processes all python -m pytest tests/test_p2p_multiprocess.py -q -x -k "2-4 and A" > gpurun_out/sanitizer_memcheck_mp.log 2>&1; echo memcheck_mp=$? >> gpurun_out/status18.txt
echo done >> gpurun_out/status18.txt
