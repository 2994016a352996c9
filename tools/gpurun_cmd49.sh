cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sim --launch-skip 2 -c 1 -o gpurun_out/r2_ksim_applies python tools/replay_paradigm.py dssp applies > gpurun_out/r2_ncu_applies.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sim --launch-skip 2 -c 1 -o gpurun_out/r2_ksim_pulls python tools/replay_paradigm.py dssp pulls > gpurun_out/r2_ncu_pulls.log 2>&1
