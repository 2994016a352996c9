#!/bin/sh
# Profiling build of the engine (globaltimer phase counters in the device run
# loop and the sharded step): tools/libdssp_ps_prof.so, used via DSSP_PS_LIB.
cd "$(dirname "$0")/../paper_1908_11848_b200/csrc" && \
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -DPS_SHARD_PROFILE -DPS_SIM_PROFILE -shared -o ../../tools/libdssp_ps_prof.so \
  ps_server.cu ps_sim.cu ps_shard.cu ps_workers.cu
