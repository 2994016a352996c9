cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_replay_gate_scan.py tests/test_gpu_acceptance.py tests/test_gpu_throttle.py -q -x 2>&1 | tail -5 > gpurun_out/r2_t56.log
{ for rep in 1 2; do for sc in 1 0; do for p in dssp asp; do for m in full data; do PS_REPLAY_GATE_SCAN=$sc timeout 120 python tools/replay_paradigm.py $p $m | sed "s|^|scan=$sc |"; done; done; done; done; } > gpurun_out/r2_dstream.txt 2>&1
