cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_replay_gate_scan.py tests/test_gpu_acceptance.py -q -x 2>&1 | tail -3 > gpurun_out/r2_t54.log
{ for rep in 1 2; do for lib in paper_1908_11848_b200/libdssp_ps.so tools/libdssp_ps_branched.so; do for nt in 128 256; do for m in full data pulls applies; do DSSP_PS_LIB=$lib PS_REPLAY_NT=$nt timeout 120 python tools/replay_paradigm.py dssp $m | sed "s|^|$(basename $lib) nt=$nt |"; done; done; done; done; } > gpurun_out/r2_straight.txt 2>&1
