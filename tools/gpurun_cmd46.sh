cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_replay.py -q -x 2>&1 | tail -3 > gpurun_out/r2_t46.log
{ for rep in 1 2; do for cv in 0 1; do for m in full data pulls applies; do if [ $cv = 1 ]; then export PS_SIM_DEFAULT_CARVEOUT=1; else unset PS_SIM_DEFAULT_CARVEOUT; fi; timeout 120 python tools/replay_paradigm.py dssp $m | sed "s/^/default_carveout=$cv /"; done; done; done; } > gpurun_out/r2_carve.txt 2>&1
