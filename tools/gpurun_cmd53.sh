cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_replay_gate_scan.py tests/test_gpu_sim.py tests/test_gpu_throttle.py tests/test_gpu_acceptance.py -q -x 2>&1 | tail -3 > gpurun_out/r2_t53.log
{ for rep in 1 2; do for nt in 128 256; do for m in full data; do PS_REPLAY_NT=$nt timeout 120 python tools/replay_paradigm.py dssp $m | sed "s/^/nt=$nt /"; done; done; done; } > gpurun_out/r2_nt2.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_b53.json 2> gpurun_out/r2_b53.err
