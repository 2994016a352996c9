cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_sharded.py -q 2>&1 | tail -5 > gpurun_out/r2_t31.log
for n in 2 4; do
timeout 300 ncu --target-processes all --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_shard_stream_probe --clock-control none --csv python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2969$n tools/shard_nvlink_probe.py > gpurun_out/r2_ncu_shard_probe_g$n.csv 2> gpurun_out/r2_ncu_shard_probe_g$n.err
done
for n in 2 4; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2979$n tools/shard_time.py 2>&1 | grep step_us; done > gpurun_out/r2_shard_time_refactor.txt
timeout 120 python tools/shard_time.py 2>&1 | grep step_us >> gpurun_out/r2_shard_time_refactor.txt
