cd $GRAFT_REPO_ROOT
{ for c in 0 120 100 80 73 60; do for m in full data; do timeout 120 python tools/replay_paradigm.py dssp $m $c; done; done; } > gpurun_out/r2_ctas.txt 2>&1
