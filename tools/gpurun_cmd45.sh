cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/replay_ceiling_probe tools/replay_ceiling_probe.cu
{ for a in "1004 1000" "1004 0" "0 1000"; do tools/replay_ceiling_probe 272474 $a; done
  for m in data pulls applies; do timeout 120 python tools/replay_paradigm.py dssp $m; done; } > gpurun_out/r2_ceiling.txt 2>&1
