cd $GRAFT_REPO_ROOT
for p in dssp ssp bsp asp; do for m in full gate data; do timeout 120 python tools/replay_paradigm.py $p $m; done; done > gpurun_out/r2_replay_split.txt 2>&1
for p in dssp asp; do DSSP_PS_LIB=tools/libdssp_ps_prof.so timeout 120 python tools/replay_paradigm.py $p full; done > gpurun_out/r2_replay_prof.txt 2>&1
timeout 300 python tools/apply_sweep_probe.py > gpurun_out/r2_apply_small2.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_replay.py -q -x 2>&1 | tail -5 > gpurun_out/r2_t16.log
