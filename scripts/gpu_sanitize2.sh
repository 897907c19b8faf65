cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
rm -f gpurun_out/status_san2.txt
S=/usr/local/cuda/bin/compute-sanitizer
K1="(synth_100_rounds_parity and 4097 and (fused or collA or collB or p2p)) or hierarchical_one_gpu or learner_step_overlapped or learner_softmax_c1 or mlp_learner_sma or learner_step_fused"
timeout 1800 $S --tool memcheck python -m pytest tests/test_gpu_parity.py -q -x -k "$K1 and not nvls" > gpurun_out/san2_memcheck.log 2>&1; echo memcheck=$? >> gpurun_out/status_san2.txt
timeout 1800 $S --tool racecheck python -m pytest tests/test_gpu_parity.py -q -x -k "(synth_100_rounds_parity and 4097 and (fused or collB)) or (hierarchical_one_gpu and (fused or p2pB)) or learner_softmax_c1" > gpurun_out/san2_racecheck.log 2>&1; echo racecheck=$? >> gpurun_out/status_san2.txt
timeout 1800 $S --tool synccheck python -m pytest tests/test_gpu_parity.py -q -x -k "(synth_100_rounds_parity and 4097 and (fused or collB)) or (hierarchical_one_gpu and (fused or p2pB)) or learner_softmax_c1" > gpurun_out/san2_synccheck.log 2>&1; echo synccheck=$? >> gpurun_out/status_san2.txt
timeout 1800 $S --tool memcheck --target-processes all python -m pytest tests/test_p2p_multiprocess.py -q -x -k "hierarchical_ranks and 2-4-None and A" > gpurun_out/san2_memcheck_mp.log 2>&1; echo memcheck_mp=$? >> gpurun_out/status_san2.txt
echo done >> gpurun_out/status_san2.txt
