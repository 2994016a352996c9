cd $GRAFT_REPO_ROOT
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29674 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2_bench_n4b.json 2> gpurun_out/r2_bench_n4b.err
