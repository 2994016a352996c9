cd $GRAFT_REPO_ROOT
run() { # tag lib ctas
  for n in 1 2 4; do
    if [ $n = 1 ]; then TAG="$1 cps=$3" DSSP_PS_LIB=$2 PS_SHARD_CTAS_PER_SM=$3 timeout 120 python tools/shard_time.py 2>&1 | grep step_us;
    else TAG="$1 cps=$3" DSSP_PS_LIB=$2 PS_SHARD_CTAS_PER_SM=$3 timeout 180 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2978$n tools/shard_time.py 2>&1 | grep step_us; fi
  done
}
{
run base paper_1908_11848_b200/libdssp_ps.so 2
run A tools/libdssp_ps_A.so 3
run B tools/libdssp_ps_B.so 2
run C tools/libdssp_ps_C.so 3
run C2 tools/libdssp_ps_C.so 2
run D tools/libdssp_ps_D.so 1
run base3 paper_1908_11848_b200/libdssp_ps.so 1
} > gpurun_out/r2_shard_variants.txt 2>&1
