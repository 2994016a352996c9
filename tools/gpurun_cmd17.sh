cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sim -c 1 -o gpurun_out/r2_ksim_replay python tools/replay_paradigm.py dssp full > gpurun_out/r2_ncu_ksim.log 2>&1
ncu -i gpurun_out/r2_ksim_replay.ncu-rep --page source --csv > gpurun_out/r2_ksim_source.csv 2>/dev/null
ncu -i gpurun_out/r2_ksim_replay.ncu-rep --page raw --csv > gpurun_out/r2_ksim_raw.csv 2>/dev/null
rm -f gpurun_out/r2_ksim_replay.ncu-rep
timeout 300 ncu --target-processes all --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_shard_run --csv python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29655 tools/shard_probe_small.py > gpurun_out/r2_ncu_shard_nvlink.csv 2> gpurun_out/r2_ncu_shard_nvlink.err
