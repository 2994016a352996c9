cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_replay_gate_scan.py tests/test_gpu_acceptance.py -q -x 2>&1 | tail -3 > gpurun_out/r2_t55.log
{ for rep in 1 2; do for lib in paper_1908_11848_b200/libdssp_ps.so tools/libdssp_ps_kg4.so; do for p in dssp asp; do for m in full data pulls applies; do DSSP_PS_LIB=$lib timeout 120 python tools/replay_paradigm.py $p $m | sed "s|^|$(basename $lib) |"; done; done; done; done; } > gpurun_out/r2_kg.txt 2>&1
