cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_sharded.py -q 2>&1 | tail -8 > gpurun_out/r2_t14.log
PS_RESIDENT=16 timeout 300 python tools/percall_probe.py > gpurun_out/r2_percall_resident2.txt 2>&1
timeout 300 python tools/shard_one.py > gpurun_out/r2_shard_one_head.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:^k_shard_run -s 1 -c 1 -o gpurun_out/r2_kshard_g1 python tools/shard_one.py > gpurun_out/r2_ncu_kshard.log 2>&1
ncu -i gpurun_out/r2_kshard_g1.ncu-rep --page raw --csv > gpurun_out/r2_kshard_g1_raw.csv 2>/dev/null
