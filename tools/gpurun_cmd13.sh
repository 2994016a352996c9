cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_server.py -q 2>&1 | tail -8 > gpurun_out/r2_t13a.log
PS_RESIDENT=16 timeout 300 python tools/percall_probe.py > gpurun_out/r2_percall_resident.txt 2>&1
PS_RESIDENT=64 timeout 300 python tools/percall_probe.py >> gpurun_out/r2_percall_resident.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_sharded.py -q 2>&1 | tail -8 > gpurun_out/r2_t13b.log
