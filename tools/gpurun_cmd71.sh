cd $GRAFT_REPO_ROOT
for L in 2 4; do DSSP_PS_LIB=tools/libdssp_ps_L$L.so timeout 600 python -m pytest tests/test_gpu_replay.py -q -x 2>&1 | tail -1 | sed "s/^/L=$L /"; done > gpurun_out/r2_t71.log
{ for rep in 1 2; do for lib in paper_1908_11848_b200/libdssp_ps.so tools/libdssp_ps_L2.so tools/libdssp_ps_L4.so; do for p in dssp asp; do for m in full data; do DSSP_PS_LIB=$lib timeout 120 python tools/replay_paradigm.py $p $m | sed "s|^|$(basename $lib) |"; done; done; done; done; } > gpurun_out/r2_lag.txt 2>&1
