cd $GRAFT_REPO_ROOT
for p in dssp asp; do for m in full data; do timeout 120 python tools/replay_paradigm.py $p $m; done; done > gpurun_out/r2_replay_split4.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_throttle.py -q -x 2>&1 | tail -5 > gpurun_out/r2_t29.log
