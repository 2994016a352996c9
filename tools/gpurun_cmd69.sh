cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_replay_gate_scan.py tests/test_gpu_acceptance.py tests/test_gpu_throttle.py -q -x 2>&1 | tail -5 > gpurun_out/r2_t69.log
{ for rep in 1 2; do for ah in 1 0; do for p in dssp ssp asp; do PS_REPLAY_CTL_AHEAD=$ah timeout 120 python tools/replay_paradigm.py $p full | sed "s|^|ahead=$ah |"; done; done; done; } > gpurun_out/r2_ahead.txt 2>&1
DSSP_PS_LIB=tools/libdssp_ps_prof.so timeout 120 python tools/replay_paradigm.py dssp full > gpurun_out/r2_ahead_prof.txt 2>&1
