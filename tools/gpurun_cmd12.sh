cd $GRAFT_REPO_ROOT
mkdir -p /tmp/sv
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29610 tests/_sharded_worker.py /tmp/sv > gpurun_out/r2_sv2.log 2>&1
cat /tmp/sv/rank0.json >> gpurun_out/r2_sv2.log 2>/dev/null
timeout 900 python -m pytest tests/test_gpu_server.py -q -x 2>&1 | tail -25 > gpurun_out/r2_t12.log
PS_RESIDENT=16 timeout 300 python tools/percall_probe.py > gpurun_out/r2_percall_resident.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_w --clock-control none --csv python tools/nvlink_probe.py 16777216 3 > gpurun_out/r2_ncu_nvlink_probe.csv 2> gpurun_out/r2_ncu_nvlink_probe.err
