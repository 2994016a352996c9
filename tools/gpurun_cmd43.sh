cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_replay_gate_scan.py -q -x 2>&1 | tail -5 > gpurun_out/r2_t43.log
{ for rep in 1 2; do for p in dssp asp; do for m in full data; do timeout 120 python tools/replay_paradigm.py $p $m; done; done; done; } > gpurun_out/r2_l1.txt 2>&1
