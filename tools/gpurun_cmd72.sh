cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sim --launch-skip 2 -c 1 -o gpurun_out/r2_ksim_c2_head python tools/replay_paradigm.py dssp full > gpurun_out/r2_ncu_c2_head.log 2>&1
