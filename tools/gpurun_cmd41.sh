cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_replay_gate_scan.py tests/test_gpu_replay.py tests/test_gpu_gate.py tests/test_gpu_sim.py -q -x 2>&1 | tail -15 > gpurun_out/r2_t41.log
{ for sc in 0 1; do for p in dssp ssp asp; do for m in full gate; do PS_REPLAY_GATE_SCAN=$sc timeout 120 python tools/replay_paradigm.py $p $m | sed "s/^/scan=$sc /"; done; done; done; } > gpurun_out/r2_scan2.txt 2>&1
