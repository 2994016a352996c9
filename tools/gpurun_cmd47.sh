cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_replay_gate_scan.py tests/test_gpu_sim.py -q -x 2>&1 | tail -3 > gpurun_out/r2_t47.log
{ for rep in 1 2; do for p in dssp asp; do for m in full data pulls applies; do timeout 120 python tools/replay_paradigm.py $p $m; done; done; done; } > gpurun_out/r2_lean.txt 2>&1
