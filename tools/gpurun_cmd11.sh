cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_sharded.py -q -x 2>&1 | tail -30 > gpurun_out/r2_t11.log
ncu --query-metrics 2>/dev/null | grep -iE "^nvl" | head -40 > gpurun_out/r2_ncu_nvl_metrics.txt
