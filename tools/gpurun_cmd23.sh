cd $GRAFT_REPO_ROOT
run() { # tag lib
  for n in 1 2; do
    if [ $n = 1 ]; then TAG="$1" DSSP_PS_LIB=$2 timeout 120 python tools/shard_time.py 2>&1 | grep step_us;
    else TAG="$1" DSSP_PS_LIB=$2 timeout 180 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2978$n tools/shard_time.py 2>&1 | grep step_us; fi
  done
}
{ for rep in 1 2; do run base paper_1908_11848_b200/libdssp_ps.so; run S1 tools/libdssp_ps_S1.so; run S2 tools/libdssp_ps_S2.so; done; } > gpurun_out/r2_shard_cache.txt 2>&1
