cd $GRAFT_REPO_ROOT
for lag in 0 1; do echo "no_lag=$lag"; PS_SHARD_NO_LAG=$lag timeout 120 python tools/shard_one.py; done > gpurun_out/r2_shard_g1_lag.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_sharded.py -q -x 2>&1 | tail -30 > gpurun_out/r2_t9.log
for n in 2 4; do for lag in 0 1; do echo "n=$n no_lag=$lag"; PS_SHARD_NO_LAG=$lag timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n bench.py --gpus $n --steps 20 --warmup 5 --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['parity'])"; done; done > gpurun_out/r2_bench_lag.txt 2>&1
