cd $GRAFT_REPO_ROOT
{ for p in dssp asp; do for m in full gate; do DSSP_PS_LIB=tools/libdssp_ps_prof.so timeout 120 python tools/replay_paradigm.py $p $m 2>&1 | tail -2; done; done; } > gpurun_out/r2_scanprof.txt 2>&1
