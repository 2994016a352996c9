cd $GRAFT_REPO_ROOT
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/push_direction_probe tools/push_direction_probe.cu
{ ./tools/push_direction_probe 23528522 2; ./tools/push_direction_probe 23528522 4; ./tools/push_direction_probe 268435456 2; ./tools/push_direction_probe 268435456 4; } > gpurun_out/r2_push_direction.txt 2>&1
