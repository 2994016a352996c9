cd $GRAFT_REPO_ROOT
for c in 1 2 3 4 6 8; do echo "ctas_per_sm=$c"; PS_SHARD_CTAS_PER_SM=$c timeout 120 python tools/shard_one.py; done > gpurun_out/r2_shard_g1_ctas.txt 2>&1
DSSP_PS_LIB=tools/libdssp_ps_prof.so timeout 120 python tools/shard_one.py > gpurun_out/r2_shard_g1_prof.txt 2>&1
