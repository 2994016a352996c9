cd $GRAFT_REPO_ROOT
PS_REPLAY_WIDE=1 timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_replay_gate_scan.py -q -x 2>&1 | tail -5 > gpurun_out/r2_t44.log
{ for rep in 1 2; do for wide in 0 1; do for p in dssp asp; do for m in full data; do PS_REPLAY_WIDE=$wide timeout 120 python tools/replay_paradigm.py $p $m | sed "s/^/wide=$wide /"; done; done; done; done; } > gpurun_out/r2_wide.txt 2>&1
