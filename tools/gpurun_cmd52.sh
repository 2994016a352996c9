cd $GRAFT_REPO_ROOT
PS_REPLAY_NT=128 timeout 600 python -m pytest tests/test_gpu_replay.py tests/test_gpu_replay_gate_scan.py -q -x 2>&1 | tail -3 > gpurun_out/r2_t52.log
{ for rep in 1 2; do for cfg in "0 2" "128 2" "128 4"; do set -- $cfg; for m in full data pulls applies; do PS_REPLAY_NT=$1 PS_REPLAY_KG4=$2 timeout 120 python tools/replay_paradigm.py dssp $m | sed "s/^/nt=$1 kg4=$2 /"; done; done; done; } > gpurun_out/r2_nt.txt 2>&1
